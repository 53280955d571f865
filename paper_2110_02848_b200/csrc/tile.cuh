// tile.cuh -- the "tile" kernels of a single large composition.  Included by
// compose.cu inside its anonymous namespace (uses Ctx, CompDev, LevelCtrl, chunk_of).
//
// A TILE is a run of consecutive pair-space rows (A states) a_0..a_{X-1} (X <= 8) whose A arcs in one
// A-role view fit in the SLOTS of a mask word M (64 for the bottom-up levels and the counts, 32 for the
// emit; slot = one A arc, plus one "self" slot per row when B's view has eps items).  For every column
// b (B state) the tile looks at the pairs (a_x, b) of all its rows at once:
//   * lm[li]  (M): the slots whose A arc matches a B item of label index li
//                  (li = 0: B's sentinel item "B stays" -> A arcs with olabel eps (M2);
//                   li = 1: eps items -> A eps arcs (M1 eps:eps) and self slots (M3);
//                   li = l + 2: label l; 255 = padding)
//   * RT[b']  (M): the slot-transposed bitmap -- bit s = vis(row of slot s, b')
//   * B items of b in an ELL tiled by words: item j of column b at [(b / 32) * wd + j][b % 32] (column
//     0 = the sentinel "b itself"), packed (li << 24 | b'); a word's items are one contiguous block
// so ONE shared load per (b, item) and an AND give the candidate moves of all X pairs into vis:
//   hits = lm[li] & RT[b'];  pair (a_x, b) has a move into vis  <=>  hits & rowmask[x] != 0.
// This is the frontier-parallel arc-pair exploration of PAPER.md:237-248 (§3.3) organised so that the
// arc-pair test is word-parallel over the A side (64 slots per AND) instead of one thread per pair.
// BYTE mode (every row of the view has <= 8 slots): row x owns slots [8x, 8x + 8), so per-row counts
// are the byte popcounts of the hit word (SWAR).
//
// Kernels:
//   k_tile_pull<false>  stage 1 bottom-up round (PAPER.md:108-111 backward BFS): an unvisited pair
//                       (~R) is claimed iff one forward move lands in R.
//   k_tile_pull<true>   stage 2 bottom-up round (Alg. 1 l.12-31, restricted to R): an unvisited pair
//                       in R \ V is claimed iff one predecessor (reversed move, in-views) is in V.
//   k_tile_count        pass-1 arc counts: kept moves per 1024-pair block / word.
//   k_tile_emit         pass 2: writes the composed CSR at scan-derived slots.

#ifndef FSTC_T_THREADS
#define FSTC_T_THREADS 1024
#endif
constexpr int kTThreads = FSTC_T_THREADS;  // count / tile-push CTAs (1 per SM: the 64-bit RT takes the smem)
#ifndef FSTC_TP1_THREADS
#define FSTC_TP1_THREADS 1024
#endif
#ifndef FSTC_TP2_THREADS
#define FSTC_TP2_THREADS 896
#endif
constexpr int kTP1Threads = FSTC_TP1_THREADS;  // stage-1 bottom-up rounds
constexpr int kTP2Threads = FSTC_TP2_THREADS;  // stage-2 rounds (fewer threads, more registers: no spills at kJ = 16)
constexpr int kTWarps = kTThreads / 32;
#ifndef FSTC_E_THREADS
#define FSTC_E_THREADS 896
#endif
constexpr int kEThreads = FSTC_E_THREADS; // emit CTAs (1 per SM: the rank tables take the shared memory)
constexpr int kEWarps = kEThreads / 32;
constexpr int kPSlots = 64;              // slots of the pull / count tiles
constexpr int kESlots = 32;              // slots of the emit tiles
constexpr int kTRows = 8;
constexpr int kTLab = 256;
constexpr uint32_t kLiSent = 0u, kLiEps = 1u, kLiPad = 255u;
constexpr int kECap = 192;               // per-warp arc-code buffer of the emit (arcs per flush)
constexpr int kTileSmemMax = 200 * 1024;
constexpr int kJReg = 16;                // ELL columns held in registers per word (more: a tail loop)

struct TileSide {
  // A-role view (slots): arcs of row a are [off[a], off[a+1])
  const int32_t* off;
  const int32_t* key;
  const int32_t* other;
  const int32_t* carry;
  const float* w;
  // B-role ELL
  const uint32_t* ell;  // [wpr][wd][32] (word-tiled ELL)
  const int2* ellcw;    // [wpr][wd][32] (carry, weight bits) of the arc behind each ELL entry (emit)
  const uint8_t* wmax;  // [wpr] ELL columns used by the 32 states of each word
  int32_t wd;
};

struct TileArgs {
  TileSide sd;
  const int32_t* trow;  // [ntiles + 1]
  int32_t ntiles;
  int32_t self;         // one self slot per row (B view has eps items)
  int32_t bytemode;     // row x owns slots [8x, 8x + 8)
  int32_t kj;           // ELL columns held in registers (template instance: 8 or 16)
  int32_t t0, t1;       // tiles [t0, t1) this launch processes (a shard: the tiles over its rows)
};

template <typename M>
struct TileSmem {
  M lm[kTLab];
  int32_t srow[8 * sizeof(M)];
  int32_t scarry[8 * sizeof(M)];
  float sw[8 * sizeof(M)];
  M rmask[kTRows];
  M selfm;
  int32_t r0, nr, ns;
};

__device__ __forceinline__ int popc_m(uint32_t x) { return __popc(x); }
__device__ __forceinline__ int popc_m(unsigned long long x) { return __popcll(x); }
__device__ __forceinline__ int ffs_m(uint32_t x) { return __ffs(x); }
__device__ __forceinline__ int ffs_m(unsigned long long x) { return __ffsll((long long)x); }

// lane i holds row i (bit j = element (i, j)); returns column `lane` (bit i = element (i, lane)).
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
#pragma unroll
  for (int k = 16; k >= 1; k >>= 1) {
    const uint32_t m = k == 16 ? 0x0000FFFFu : k == 8 ? 0x00FF00FFu : k == 4 ? 0x0F0F0F0Fu : k == 2 ? 0x33333333u : 0x55555555u;
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, k);
    x = (lane & k) ? ((x & ~m) | ((y >> k) & m)) : ((x & m) | ((y << k) & ~m));
  }
  return x;
}

// Slots and label masks of tile `tile` (all threads; two barriers).  Warp 0 lays out the rows' slot
// ranges; then one thread per slot loads its arc (one round of independent loads, not a chain).
template <typename M>
__device__ void tile_slots(TileSmem<M>& t, const TileArgs& ta, int tile) {
  constexpr int kS = 8 * sizeof(M);
  __shared__ int32_t s_e0[kTRows], s_s0[kTRows], s_d[kTRows];
  for (int i = threadIdx.x; i < kTLab; i += blockDim.x) t.lm[i] = M(0);
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const int32_t r0 = __ldg(&ta.trow[tile]), r1 = __ldg(&ta.trow[tile + 1]);
    const int nr = r1 - r0;
    int32_t e0 = 0, d = 0;
    if (lane < nr) {
      e0 = __ldg(&ta.sd.off[r0 + lane]);
      d = __ldg(&ta.sd.off[r0 + lane + 1]) - e0;
    }
    const int n = lane < nr ? d + ta.self : 0;
    int s0, ns;
    if (ta.bytemode) {
      s0 = 8 * lane;
      ns = 8 * nr;
    } else {
      const int inc = warp_incl_scan(n);
      s0 = inc - n;
      ns = __shfl_sync(0xffffffffu, inc, 31);
    }
    M self = M(0);
    if (lane < nr) {
      t.rmask[lane] = n >= kS ? ~M(0) : (((M(1) << n) - M(1)) << s0);
      s_e0[lane] = e0;
      s_s0[lane] = s0;
      s_d[lane] = d;
      if (ta.self) {
        t.srow[s0] = r0 + lane;
        t.scarry[s0] = FST_EPS;
        t.sw[s0] = 0.f;
        self = M(1) << s0;
      }
    }
    // OR of the self-slot bits over the rows (warp reduction)
    unsigned long long sm64 = (unsigned long long)self;
#pragma unroll
    for (int k = 16; k > 0; k >>= 1) sm64 |= __shfl_xor_sync(0xffffffffu, sm64, k);
    if (lane == 0) {
      t.r0 = r0;
      t.nr = nr;
      t.ns = ns;
      t.selfm = (M)sm64;
    }
  }
  __syncthreads();
  const int nr = t.nr;
  // label-mask bits via 32-bit shared atomics (a 64-bit shared atomicOr is a CAS loop)
  auto lm_or = [&](int li, int s) { atomicOr((uint32_t*)&t.lm[li] + (s >> 5), 1u << (s & 31)); };
  if (ta.self && threadIdx.x < 32 && threadIdx.x < nr) lm_or(kLiEps, s_s0[threadIdx.x]);  // M3: B eps item, A stays
  // one thread per (row, arc): slot s0_x + self + k
  for (int i = threadIdx.x; i < nr * kS; i += blockDim.x) {
    const int x = i / kS, k = i - x * kS;
    if (k >= s_d[x]) continue;
    const int32_t e = s_e0[x] + k;
    const int s = s_s0[x] + ta.self + k;
    const int32_t l = __ldg(&ta.sd.key[e]);
    t.srow[s] = __ldg(&ta.sd.other[e]);
    t.scarry[s] = __ldg(&ta.sd.carry[e]);
    t.sw[s] = __ldg(&ta.sd.w[e]);
    lm_or(l + 2, s);                     // M1 (eps:eps included: l = -1 -> 1)
    if (l == FST_EPS) lm_or(kLiSent, s);  // M2: A eps arc, B stays (sentinel)
  }
  if (ta.bytemode) {  // unused slots of byte mode: any valid row (they are in no label mask)
    for (int s = threadIdx.x; s < t.ns; s += blockDim.x) {
      const int x = s >> 3, k = (s & 7) - ta.self;
      if ((s & 7) >= s_d[x] + ta.self) t.srow[s] = t.r0;
      (void)k;
    }
  }
  __syncthreads();
}

// RT[b'] = bits over slots s of vis(srow[s], b'), for all columns (all threads; no barrier).  Each
// warp issues the loads of 4 words before transposing them.
__device__ __forceinline__ void tile_rt(uint32_t* RT, const TileSmem<uint32_t>& t, const uint32_t* __restrict__ vis,
                                        int64_t W, int wpr, int nwarps) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t* rowp = lane < t.ns ? vis + W + (int64_t)t.srow[lane] * wpr : nullptr;
  for (int w0 = warp; w0 < wpr; w0 += 4 * nwarps) {
    uint32_t x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int w = w0 + u * nwarps;
      x[u] = (rowp && w < wpr) ? __ldg(rowp + w) : 0u;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int w = w0 + u * nwarps;
      const uint32_t c = transpose32(x[u], lane);
      if (w < wpr) RT[w * 32 + lane] = c;
    }
  }
}
__device__ __forceinline__ void tile_rt(unsigned long long* RT, const TileSmem<unsigned long long>& t,
                                        const uint32_t* vis, int64_t W, int wpr, int nwarps) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t* rp0 = lane < t.ns ? vis + W + (int64_t)t.srow[lane] * wpr : nullptr;
  const uint32_t* rp1 = lane + 32 < t.ns ? vis + W + (int64_t)t.srow[lane + 32] * wpr : nullptr;
  for (int w0 = warp; w0 < wpr; w0 += 2 * nwarps) {
    uint32_t x[4];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int w = w0 + u * nwarps;
      x[2 * u] = (rp0 && w < wpr) ? __ldca(rp0 + w) : 0u;  // (L1-cached; a stale word only delays a claim)
      x[2 * u + 1] = (rp1 && w < wpr) ? __ldca(rp1 + w) : 0u;
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int w = w0 + u * nwarps;
      const uint32_t lo = transpose32(x[2 * u], lane), hi = transpose32(x[2 * u + 1], lane);
      if (w < wpr) RT[w * 32 + lane] = ((unsigned long long)hi << 32) | lo;
    }
  }
}

// Ring bookkeeping of a level that runs on tile kernels (the same as k_level's block-0 prologue).
__device__ __forceinline__ void tile_level_prologue(const Ctx& cx, int level) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    LevelCtrl* ctrl_cur = &cx.ctrl[level % 3];
    LevelCtrl* ctrl_nxt = &cx.ctrl[(level + 1) % 3];
    LevelCtrl* z = &cx.ctrl[(level + 2) % 3];
    z->count = 0;
    z->nnew = 0;
    cx.misc[0] += 1;
    if (level < kMaxLevelStats) cx.hist[level] = ctrl_cur->nnew;
    ctrl_nxt->pad[0] = ctrl_cur->pad[0] + ctrl_cur->nnew;
  }
}

// Fields of the (single) composition the tile kernels use, hoisted into registers (the kernels store
// to global memory, so reads through cx.comps would be repeated after every store).
struct TC {
  int64_t W, K, Q;
  int32_t wpr, VB, bpr, VA, cpr, CB;
  int32_t r0, r1;  // rows this rank owns (all rows unless sharded; the tile path shards by row ranges)
  __device__ __forceinline__ bool own(int32_t row) const { return row >= r0 && row < r1; }
};
__device__ __forceinline__ TC tc_of(const Ctx& cx) {
  const CompDev& C = cx.comps[0];
  const bool sh = C.sh_world > 1;
  return TC{C.W, C.K, C.Q, C.wpr, C.VB, C.bpr, C.VA, C.cpr, C.CB, sh ? C.sh_r0 : 0, sh ? C.sh_r1 : C.VA};
}

// Items of column b = 32 w + lane (ELL columns 1..jn-1; column 0, the sentinel, when j0 == 0): the
// first kJ columns are loaded together into registers (immediate offsets inside the word's block),
// the rest (rare) in a tail loop.  f(x) per item.
template <int kJ, typename F>
__device__ __forceinline__ void for_items(const uint32_t* __restrict__ ell, int wd, int w, int lane, int j0, int jn,
                                          F&& f) {
  const uint32_t* p = ell + (size_t)w * wd * 32 + lane;
  if (j0 == 0) f(__ldg(p));
  uint32_t it[kJ];
#pragma unroll
  for (int k = 0; k < kJ; ++k) it[k] = (k + 1 < jn) ? __ldg(p + (k + 1) * 32) : (kLiPad << 24);
#pragma unroll
  for (int k = 0; k < kJ; ++k) f(it[k]);
  for (int j = kJ + 1; j < jn; ++j) f(__ldg(p + j * 32));
}

// ------------------------------------------------------------------------------ bottom-up round
// One bottom-up round, IN PLACE: an unvisited pair of the tile's rows whose move set hits vis is
// claimed (vis |= new, next frontier |= new) right away, so tiles staged later in the same round see it
// and a round can claim pairs several BFS distances deep.  R and V are sets (Alg. 1 line 3; the
// forward closure restricted to R): claiming a pair as soon as one move reaches the set is sound, and
// the stage loop runs until a round claims nothing (the fixed point), so the sets are exact.  Only the
// per-round sizes differ from per-BFS-distance counts.  Each tile also consumes the current frontier
// words and chunk flags of its rows and lists the chunks that gained next-frontier bits (for a
// following push level), so no separate merge pass is needed.
template <bool kStage2, int kJ, int NT>
__global__ void __launch_bounds__(NT, 1) k_tile_pull(Ctx cx, TileArgs ta, int level) {
  using M = unsigned long long;
  __shared__ TileSmem<M> t;
  __shared__ uint32_t chit[kTRows][2];  // per tile row: chunks (<= 64) that gained next-frontier bits
  __shared__ int s_any;
  extern __shared__ __align__(16) unsigned long long tdyn64[];
  M* RT = tdyn64;
  tile_level_prologue(cx, level);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const TC c = tc_of(cx);
  uint32_t* vis = kStage2 ? cx.V : cx.R;   // read and written in place (plain loads: other CTAs write it)
  const uint32_t* __restrict__ Rb = cx.R;  // stage 2: R is fixed
  const int p = level & 1;
  uint32_t* Fc = p ? cx.F1 : cx.F0;
  uint32_t* Fn = p ? cx.F0 : cx.F1;
  uint32_t* flagc = p ? cx.flag1 : cx.flag0;
  uint32_t* flagn = p ? cx.flag0 : cx.flag1;
  int32_t* listn = p ? cx.list0 : cx.list1;
  LevelCtrl* ctrl_nxt = &cx.ctrl[(level + 1) % 3];
  const uint32_t* __restrict__ ell = ta.sd.ell;
  const uint8_t* __restrict__ wmax = ta.sd.wmax;
  const int wpr = c.wpr, VB = c.VB;
  const uint32_t lastmask = (VB & 31) ? (1u << (VB & 31)) - 1u : ~0u;
  auto unvisited = [&](int32_t row, int w) -> uint32_t {  // (0 for rows of other shards)
    if (!c.own(row)) return 0u;
    const int64_t gw = c.W + (int64_t)row * wpr + w;
    const uint32_t v = __ldca(&vis[gw]);
    uint32_t u = kStage2 ? (__ldg(&Rb[gw]) & ~v) : ~v;
    return w == wpr - 1 ? (u & lastmask) : u;
  };
  unsigned nnew = 0;
  for (int tile = ta.t0 + blockIdx.x; tile < ta.t1; tile += gridDim.x) {
    tile_slots(t, ta, tile);
    const int nr = t.nr;
    const int32_t r0 = t.r0;
    if (threadIdx.x < 2 * kTRows) chit[threadIdx.x >> 1][threadIdx.x & 1] = 0u;
    if (threadIdx.x == 0) s_any = 0;
    __syncthreads();
    // consume the rows' frontier words; any unvisited pair left?
    bool any = false;
    for (int i = threadIdx.x; i < nr * wpr; i += NT) {
      const int x = i / wpr, w = i - x * wpr;
      const int64_t gw = c.W + (int64_t)(r0 + x) * wpr + w;
      if (Fc[gw]) Fc[gw] = 0u;
      any |= unvisited(r0 + x, w) != 0u;
    }
    if (any) s_any = 1;
    __syncthreads();
    if (s_any) {
      tile_rt(RT, t, vis, c.W, wpr, (NT / 32));
      __syncthreads();
      const int j0 = t.lm[kLiSent] ? 0 : 1;  // the sentinel column only matters with A eps arcs
      M rm[kTRows];
#pragma unroll
      for (int x = 0; x < kTRows; ++x) rm[x] = x < nr ? t.rmask[x] : M(0);
      const M* lm = t.lm;
      // two words per warp iteration: both words' item loads are in flight together
      auto claim = [&](int w, uint32_t u, M acc) {
        uint32_t mine = 0u;
#pragma unroll
        for (int x = 0; x < kTRows; ++x) {
          if (x >= nr) break;
          const uint32_t ux = __shfl_sync(0xffffffffu, u, x);
          const uint32_t nb = __ballot_sync(0xffffffffu, (acc & rm[x]) != M(0)) & ux;
          if (lane == x) mine = nb;
        }
        if (mine) {  // lane x: claim the new pairs of (row x, w) in place
          const int64_t gw = c.W + (int64_t)(r0 + lane) * wpr + w;
          vis[gw] = __ldca(&vis[gw]) | mine;  // only this tile writes its rows
          Fn[gw] = mine;
          nnew += __popc(mine);
          const int qj = (w >> 5) / c.CB;
          atomicOr(&chit[lane][qj >> 5], 1u << (qj & 31));
        }
      };
      const int wd = ta.sd.wd;
      for (int w = warp; w < wpr; w += 2 * (NT / 32)) {
        const int w2 = w + (NT / 32);
        const uint32_t u1 = lane < nr ? unvisited(r0 + lane, w) : 0u;
        const uint32_t u2 = (w2 < wpr && lane < nr) ? unvisited(r0 + lane, w2) : 0u;
        const bool a1 = __any_sync(0xffffffffu, u1 != 0u), a2 = __any_sync(0xffffffffu, u2 != 0u);
        if (!a1 && !a2) continue;
        const int b1 = w * 32 + lane, b2 = w2 * 32 + lane;
        const bool v1 = a1 && b1 < VB, v2 = a2 && b2 < VB;
        const int jn1 = v1 ? wmax[w] : 0, jn2 = v2 ? wmax[w2] : 0;
        const uint32_t* p1 = ell + (size_t)w * wd * 32 + lane;
        const uint32_t* p2 = ell + (size_t)w2 * wd * 32 + lane;
        uint32_t i1[kJ], i2[kJ];
#pragma unroll
        for (int k = 0; k < kJ; ++k) {
          i1[k] = (k + 1 < jn1) ? __ldg(p1 + (k + 1) * 32) : (kLiPad << 24);
          i2[k] = (k + 1 < jn2) ? __ldg(p2 + (k + 1) * 32) : (kLiPad << 24);
        }
        M acc1 = M(0), acc2 = M(0);
        if (j0 == 0) {
          if (v1) { const uint32_t x = __ldg(p1); acc1 |= lm[x >> 24] & RT[x & 0xFFFFFFu]; }
          if (v2) { const uint32_t x = __ldg(p2); acc2 |= lm[x >> 24] & RT[x & 0xFFFFFFu]; }
        }
#pragma unroll
        for (int k = 0; k < kJ; ++k) {
          acc1 |= lm[i1[k] >> 24] & RT[i1[k] & 0xFFFFFFu];
          acc2 |= lm[i2[k] >> 24] & RT[i2[k] & 0xFFFFFFu];
        }
        for (int j = kJ + 1; j < jn1; ++j) { const uint32_t x = __ldg(p1 + j * 32); acc1 |= lm[x >> 24] & RT[x & 0xFFFFFFu]; }
        for (int j = kJ + 1; j < jn2; ++j) { const uint32_t x = __ldg(p2 + j * 32); acc2 |= lm[x >> 24] & RT[x & 0xFFFFFFu]; }
        if (a1) claim(w, u1, acc1);
        if (a2) claim(w2, u2, acc2);
      }
    }
    __syncthreads();
    // chunk flags of the tile's rows: consumed ones cleared, chunks with new bits listed
    for (int i = threadIdx.x; i < nr * c.cpr; i += NT) {
      const int x = i / c.cpr, j = i - x * c.cpr;
      if (!c.own(r0 + x)) continue;
      const int64_t q = c.Q + (int64_t)(r0 + x) * c.cpr + j;
      if (flagc[q]) flagc[q] = 0u;
      if ((chit[x][j >> 5] >> (j & 31)) & 1u) {
        flagn[q] = 1u;
        const unsigned long long pos = atomicAdd(&ctrl_nxt->count, 1ull);
        listn[pos] = (int32_t)q;
      }
    }
    __syncthreads();
  }
  nnew = warp_sum(nnew);
  if (lane == 0 && nnew) atomicAdd(&ctrl_nxt->nnew, (unsigned long long)nnew);
}

// ------------------------------------------------------------------------------ push level (tile form)
// A frontier-synchronous level (Alg. 1's rounds) over the tiles that hold frontier
// pairs: for a frontier pair (a_x, b) the moves out of it are lm[li] & rowmask[x] over b's items, and
// the claimable targets are the bits of RT_C = (stage 1: ~R | stage 2: R & ~V) of the slot rows; each
// target is claimed by a global test-and-set and joins the next frontier (chunk flags / lists as in
// k_level).  Stage 1 walks the reversed moves (tiles over A's in-view, B's in-item ELL), stage 2 the
// forward moves (A's out-view, B's out-items).  Tiles without frontier pairs are skipped before any
// staging, so sparse levels cost about one read of the frontier bitmap.
template <bool kStage2, int kJ>
__global__ void __launch_bounds__(kTThreads, 1) k_tile_push(Ctx cx, TileArgs ta, int level) {
  using M = unsigned long long;
  __shared__ TileSmem<M> t;
  __shared__ int s_any;
  extern __shared__ __align__(16) unsigned long long tdyn64[];
  M* RT = tdyn64;
  const TC c = tc_of(cx);
  const int wpr = c.wpr, VB = c.VB;
  uint32_t* FW = (uint32_t*)(tdyn64 + (size_t)wpr * 32);  // [kTRows][wpr] the tile's frontier words
  tile_level_prologue(cx, level);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* vis = kStage2 ? cx.V : cx.R;
  const uint32_t* __restrict__ Rb = cx.R;
  const int p = level & 1;
  uint32_t* Fc = p ? cx.F1 : cx.F0;
  uint32_t* Fn = p ? cx.F0 : cx.F1;
  uint32_t* flagc = p ? cx.flag1 : cx.flag0;
  uint32_t* flagn = p ? cx.flag0 : cx.flag1;
  int32_t* listn = p ? cx.list0 : cx.list1;
  LevelCtrl* ctrl_nxt = &cx.ctrl[(level + 1) % 3];
  const CompDev& C = cx.comps[0];
  const uint32_t* __restrict__ ell = ta.sd.ell;
  const uint8_t* __restrict__ wmax = ta.sd.wmax;
  const uint32_t lastmask = (VB & 31) ? (1u << (VB & 31)) - 1u : ~0u;
  unsigned nnew = 0;
  for (int tile = ta.t0 + blockIdx.x; tile < ta.t1; tile += gridDim.x) {
    // the rows' frontier words (consumed) -> FW; skip tiles without frontier pairs
    const int32_t r0 = __ldg(&ta.trow[tile]), nr = __ldg(&ta.trow[tile + 1]) - r0;
    if (threadIdx.x == 0) s_any = 0;
    __syncthreads();
    bool any = false;
    for (int i = threadIdx.x; i < nr * wpr; i += kTThreads) {
      const int x = i / wpr, w = i - x * wpr;
      uint32_t f = 0u;
      if (c.own(r0 + x)) {
        const int64_t gw = c.W + (int64_t)(r0 + x) * wpr + w;
        f = Fc[gw];
        if (f) Fc[gw] = 0u;
      }
      FW[x * wpr + w] = f;
      any |= f != 0u;
    }
    for (int i = threadIdx.x; i < nr * c.cpr; i += kTThreads) {  // consumed chunk flags
      const int x = i / c.cpr;
      if (!c.own(r0 + x)) continue;
      const int64_t q = c.Q + (int64_t)(r0 + x) * c.cpr + (i - x * c.cpr);
      if (flagc[q]) flagc[q] = 0u;
    }
    if (any) s_any = 1;
    __syncthreads();
    if (!s_any) continue;
    tile_slots(t, ta, tile);
    // RT_C: claimable bits of the slot rows
    {
      const uint32_t* rp0 = lane < t.ns ? vis + c.W + (int64_t)t.srow[lane] * wpr : nullptr;
      const uint32_t* rq0 = lane < t.ns ? Rb + c.W + (int64_t)t.srow[lane] * wpr : nullptr;
      const uint32_t* rp1 = lane + 32 < t.ns ? vis + c.W + (int64_t)t.srow[lane + 32] * wpr : nullptr;
      const uint32_t* rq1 = lane + 32 < t.ns ? Rb + c.W + (int64_t)t.srow[lane + 32] * wpr : nullptr;
      for (int w = warp; w < wpr; w += kTWarps) {
        const uint32_t mk = w == wpr - 1 ? lastmask : ~0u;
        uint32_t x0 = 0u, x1 = 0u;
        if (rp0) x0 = (kStage2 ? (__ldg(rq0 + w) & ~__ldca(rp0 + w)) : ~__ldca(rp0 + w)) & mk;
        if (rp1) x1 = (kStage2 ? (__ldg(rq1 + w) & ~__ldca(rp1 + w)) : ~__ldca(rp1 + w)) & mk;
        const uint32_t lo = transpose32(x0, lane), hi = transpose32(x1, lane);
        RT[w * 32 + lane] = ((unsigned long long)hi << 32) | lo;
      }
    }
    __syncthreads();
    const int j0 = t.lm[kLiSent] ? 0 : 1;
    const M* lm = t.lm;
    for (int w = warp; w < wpr; w += kTWarps) {
      const uint32_t fl = lane < nr ? FW[lane * wpr + w] : 0u;
      if (!__any_sync(0xffffffffu, fl != 0u)) continue;
      const int b = w * 32 + lane;
      const int jn = wmax[w];
      // rows x whose pair (x, b) is in the frontier, as a per-lane bit set (usually 0 or 1 rows)
      unsigned rows = 0u;
#pragma unroll
      for (int x = 0; x < kTRows; ++x) {
        const uint32_t fx = __shfl_sync(0xffffffffu, fl, x);
        if (x < nr && ((fx >> lane) & 1u) && b < VB) rows |= 1u << x;
      }
#pragma unroll 1
      while (rows) {  // (not unrolled: one copy of the item loop)
        const int x = __ffs(rows) - 1;
        rows &= rows - 1u;
        const M rmx = t.rmask[x];
        for_items<kJ>(ell, ta.sd.wd, w, lane, j0, jn, [&](uint32_t it) {
          M h = lm[it >> 24] & rmx;
          if (!h) return;
          const uint32_t o = it & 0xFFFFFFu;
          h &= RT[o];
          while (h) {  // fire-and-forget claims (RT_C excludes every pair of an earlier level)
            const int s = __ffsll((long long)h) - 1;
            h &= h - 1ull;
            const int32_t row = t.srow[s];
            const int64_t gw = c.W + (int64_t)row * wpr + (o >> 5);
            const uint32_t bit = 1u << (o & 31);
            if (!owned(C, row, (int32_t)o)) {  // sharded: the owner claims it after the exchange
              atomicOr(&cx.OUT[gw], bit);
              continue;
            }
            atomicOr(&vis[gw], bit);
            atomicOr(&Fn[gw], bit);
          }
        });
      }
    }
    __syncthreads();
  }
  (void)nnew;
  (void)flagn;
  (void)listn;
  (void)ctrl_nxt;
}

// ------------------------------------------------------------------------------ sparse push level
// A push level for small frontiers (the levels before and after the bottom-up rounds): one warp per
// active chunk (row a, <= 1024 words) from the level's list.  The warp stages the row's A arcs of the
// level's direction (stage 1: in-arcs = reversed moves, stage 2: out-arcs) as label masks over <= 64
// slots; each lane takes frontier words of the chunk and, per frontier pair (a, b), walks b's items in
// B's word-tiled ELL: a target (row of slot s, b') is claimed when its vis bit is clear -- a plain
// load, then fire-and-forget reductions on vis and the next frontier (every pair of an earlier level
// has its bit set, so the next frontier gets exactly this level's new pairs; duplicates are ORs).
// k_push_finish then counts the next frontier and lists its chunks.
constexpr int kSPLab = 64;  // label-mask entries staged per warp (label index < 64; else the tile rounds' k_level)
#ifndef FSTC_SP_MINB
#define FSTC_SP_MINB 0
#endif
#ifndef FSTC_SP_GRID
#define FSTC_SP_GRID 16
#endif
constexpr int kSPGrid = FSTC_SP_GRID;  // CTAs per SM of the push levels
template <bool kStage2>
__global__ void __launch_bounds__(256, FSTC_SP_MINB) k_sparse_push(Ctx cx, TileArgs ta, int level) {
  __shared__ unsigned long long lmw[8][kSPLab];
  __shared__ int32_t sroww[8][64];
  tile_level_prologue(cx, level);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int p = level & 1;
  uint32_t* Fc = p ? cx.F1 : cx.F0;
  uint32_t* Fn = p ? cx.F0 : cx.F1;
  uint32_t* flagc = p ? cx.flag1 : cx.flag0;
  const int32_t* listc = p ? cx.list1 : cx.list0;
  uint32_t* vis = kStage2 ? cx.V : cx.R;
  const uint32_t* __restrict__ Rb = cx.R;
  const CompDev& C = cx.comps[0];
  const TC c = tc_of(cx);
  const int wpr = c.wpr, VB = c.VB, wd = ta.sd.wd;
  const unsigned long long nlist = *((volatile unsigned long long*)&cx.ctrl[level % 3].count);
  unsigned long long* lm = lmw[wib];
  int32_t* srow = sroww[wib];
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t e = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; e < (int64_t)nlist; e += nwarps) {
    const int64_t q = listc[e];
    const int32_t row = (int32_t)((q - c.Q) / c.cpr), jc = (int32_t)(q - c.Q - (int64_t)row * c.cpr);
    if (lane == 0) flagc[q] = 0u;
    // the row's slots: self slot (when B has eps items) then its arcs
    const int32_t e0 = __ldg(&ta.sd.off[row]), d = __ldg(&ta.sd.off[row + 1]) - e0;
    for (int i = lane; i < kSPLab; i += 32) lm[i] = 0ull;
    __syncwarp();
    const int self = ta.self;
    if (self && lane == 0) {
      srow[0] = row;
      atomicOr((uint32_t*)&lm[kLiEps], 1u);  // M3
    }
    for (int k = lane; k < d; k += 32) {
      const int s = self + k;
      const int32_t l = __ldg(&ta.sd.key[e0 + k]);
      srow[s] = __ldg(&ta.sd.other[e0 + k]);
      atomicOr((uint32_t*)&lm[l + 2] + (s >> 5), 1u << (s & 31));
      if (l == FST_EPS) atomicOr((uint32_t*)&lm[kLiSent] + (s >> 5), 1u << (s & 31));
    }
    __syncwarp();
    const bool sent = lm[kLiSent] != 0ull;
    const int w0 = jc * c.CB * 32, w1 = min(w0 + c.CB * 32, wpr);
    const int64_t rw = c.W + (int64_t)row * wpr;
    for (int w = w0 + lane; w < w1; w += 32) {
      uint32_t f = Fc[rw + w];
      if (!f) continue;
      Fc[rw + w] = 0u;
      const int jn = ta.sd.wmax[w];
      const uint32_t* pb = ta.sd.ell + (size_t)w * wd * 32;
      while (f) {
        const int bb = __ffs(f) - 1;
        f &= f - 1u;
        if (w * 32 + bb >= VB) continue;
        for (int j = sent ? 0 : 1; j < jn; ++j) {
          const uint32_t it = __ldg(pb + j * 32 + bb);
          const uint32_t li = it >> 24;
          if (li >= (uint32_t)kSPLab) continue;
          unsigned long long m = lm[li];
          const uint32_t o = it & 0xFFFFFFu;
          while (m) {
            const int s = __ffsll((long long)m) - 1;
            m &= m - 1ull;
            const int32_t tr = srow[s];
            const int64_t gw = c.W + (int64_t)tr * wpr + (o >> 5);
            const uint32_t bit = 1u << (o & 31);
            if (kStage2 && !(__ldg(&Rb[gw]) & bit)) continue;  // stage 2: only pairs of R
            if (!owned(C, tr, (int32_t)o)) {                    // sharded: the owner claims it
              atomicOr(&cx.OUT[gw], bit);
              continue;
            }
            if (__ldca(&vis[gw]) & bit) continue;
            atomicOr(&vis[gw], bit);
            atomicOr(&Fn[gw], bit);
          }
        }
      }
    }
    __syncwarp();
  }
}

// After a tile push level: the next frontier's size and its chunk list (one warp per chunk; the
// push kernel's claims are plain reductions, so the exact count comes from the bitmap).
__global__ void k_push_finish(Ctx cx, int level) {
  const int p = level & 1;
  const uint32_t* Fn = p ? cx.F0 : cx.F1;
  uint32_t* flagn = p ? cx.flag0 : cx.flag1;
  int32_t* listn = p ? cx.list0 : cx.list1;
  LevelCtrl* ctrl_nxt = &cx.ctrl[(level + 1) % 3];
  const int lane = threadIdx.x & 31;
  const TC c = tc_of(cx);
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  unsigned nnew = 0;
  for (int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < cx.nchunks; q += nw) {
    const int32_t row = (int32_t)(q / c.cpr), j = (int32_t)(q - (int64_t)row * c.cpr);
    const int w0 = j * c.CB * 32, w1 = min(w0 + c.CB * 32, c.wpr);
    const int64_t rw = c.W + (int64_t)row * c.wpr;
    unsigned cnt = 0;
    for (int w = w0 + lane; w < w1; w += 32) cnt += __popc(Fn[rw + w]);
    if (__any_sync(0xffffffffu, cnt != 0u) && lane == 0) {
      flagn[q] = 1u;
      const unsigned long long pos = atomicAdd(&ctrl_nxt->count, 1ull);
      listn[pos] = (int32_t)q;
    }
    nnew += cnt;
  }
  nnew = warp_sum(nnew);
  if (lane == 0 && nnew) atomicAdd(&ctrl_nxt->nnew, (unsigned long long)nnew);
}

// ------------------------------------------------------------------------------ pass 1: counts
// kept[block] = number of moves out of the block's states of C (their out-degrees), OVERWRITTEN
// for every block of the composition, and warc[word] = the same per word (the emit's offsets).
// Tested against V (for a state of C, dst in R <=> dst in V).  Byte mode: per-row counts are SWAR
// byte popcounts of the hit words (kByte).
template <bool kByte, int kJ>
__global__ void __launch_bounds__(kTThreads, 1) k_tile_count(Ctx cx, TileArgs ta) {
  using M = unsigned long long;
  __shared__ TileSmem<M> t;
  extern __shared__ __align__(16) unsigned long long tdyn64[];
  const TC c = tc_of(cx);
  const int wpr = c.wpr, VB = c.VB, bpr = c.bpr;
  M* RT = tdyn64;
  unsigned long long* kacc = tdyn64 + (size_t)wpr * 32;  // [kTRows][bpr]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t* __restrict__ V = cx.V;
  const uint32_t* __restrict__ ell = ta.sd.ell;
  const uint8_t* __restrict__ wmax = ta.sd.wmax;
  uint32_t* warc = cx.warc;
  for (int tile = ta.t0 + blockIdx.x; tile < ta.t1; tile += gridDim.x) {
    tile_slots(t, ta, tile);
    const int nr = t.nr;
    const int32_t r0 = t.r0;
    for (int i = threadIdx.x; i < kTRows * bpr; i += kTThreads) kacc[i] = 0ull;
    tile_rt(RT, t, V, c.W, wpr, kTWarps);
    __syncthreads();
    const int j0 = t.lm[kLiSent] ? 0 : 1;
    M rm[kTRows];
#pragma unroll
    for (int x = 0; x < kTRows; ++x) rm[x] = x < nr ? t.rmask[x] : M(0);
    const M* lm = t.lm;
    // warp task: a quarter of one block (8 words)
    for (int task = warp; task < bpr * 4; task += kTWarps) {
      const int jb = task >> 2;
      const int w0 = jb * 32 + (task & 3) * 8, w1 = min(w0 + 8, wpr);
      uint32_t sums[kTRows];
#pragma unroll
      for (int x = 0; x < kTRows; ++x) sums[x] = 0u;
      const bool ownl = lane < nr && c.own(r0 + lane);  // (other shards' rows count 0 here)
      uint32_t sv = (w0 < w1 && ownl) ? __ldg(&V[c.W + (int64_t)(r0 + lane) * wpr + w0]) : 0u;
      for (int w = w0; w < w1; ++w) {
        const uint32_t svn = (w + 1 < w1 && ownl) ? __ldg(&V[c.W + (int64_t)(r0 + lane) * wpr + w + 1]) : 0u;
        uint32_t wc = 0u;  // lane x < nr: arcs of the states (row x, word w)
        if (__any_sync(0xffffffffu, sv != 0u)) {
          const int b = w * 32 + lane;
          uint32_t cr[kTRows];
#pragma unroll
          for (int x = 0; x < kTRows; ++x) cr[x] = 0u;
          if (b < VB) {
            if (kByte) {
              M bc = 0ull;  // 8 byte counters (row x = byte x); <= 31 items x 8 slots < 256
              for_items<kJ>(ell, ta.sd.wd, w, lane, j0, wmax[w], [&](uint32_t x) {
                const M h = lm[x >> 24] & RT[x & 0xFFFFFFu];
                M v = h - ((h >> 1) & 0x5555555555555555ull);
                v = (v & 0x3333333333333333ull) + ((v >> 2) & 0x3333333333333333ull);
                bc += (v + (v >> 4)) & 0x0F0F0F0F0F0F0F0Full;
              });
#pragma unroll
              for (int x = 0; x < kTRows; ++x) cr[x] = (uint32_t)(bc >> (8 * x)) & 0xFFu;
            } else {
              for_items<kJ>(ell, ta.sd.wd, w, lane, j0, wmax[w], [&](uint32_t x) {
                const M h = lm[x >> 24] & RT[x & 0xFFFFFFu];
#pragma unroll
                for (int r = 0; r < kTRows; ++r) cr[r] += __popcll(h & rm[r]);
              });
            }
          }
#pragma unroll
          for (int x = 0; x < kTRows; ++x) {
            if (x >= nr) break;
            const uint32_t sx = __shfl_sync(0xffffffffu, sv, x);
            const uint32_t cx_ = ((sx >> lane) & 1u) ? cr[x] : 0u;
            const uint32_t ws = warp_sum(cx_);
            sums[x] += ws;
            if (lane == x) wc = ws;
          }
        }
        if (ownl) warc[c.W + (int64_t)(r0 + lane) * wpr + w] = wc;
        sv = svn;
      }
#pragma unroll
      for (int x = 0; x < kTRows; ++x) {
        if (x >= nr) break;
        if (lane == 0 && sums[x]) atomicAdd(&kacc[x * bpr + jb], (unsigned long long)sums[x]);
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nr * bpr; i += kTThreads) {
      const int x = i / bpr, jb = i - x * bpr;
      if (c.own(r0 + x)) cx.kept[c.K + (int64_t)(r0 + x) * bpr + jb] = kacc[x * bpr + jb];
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------ pass 2: emit
// Output / flag arrays of the composition, passed by value (constant bank, no registers).
struct EmitIO {
  int64_t* row_ptr;
  int32_t* dst;
  int32_t* ilabel;
  int32_t* olabel;
  float* weight;
  int32_t* pair_a;
  int32_t* pair_b;
  uint8_t* is_start;
  uint8_t* is_accept;
  const uint8_t* startA;
  const uint8_t* accA;
  const uint8_t* startB;
  const uint8_t* accB;
};

// Shared memory: RT (32-bit slot-transposed V of the tile's slot rows, for the hit tests), and for
// the slot rows (the A-arc destinations, ns <= vr_rows) the V words (u32) and the rank of each word's
// first pair inside its row (u16), + per-slot-row base ids; per warp a buffer of kECap arc codes
// (dst column << 15 | item << 10 | lane << 5 | slot).  The source rows' words come from global memory
// (one load per lane and word), so the staged rows are slot rows only.
// One warp task = one word w (32 columns) for ALL rows of the tile: the word's ELL items are loaded
// once into registers and their hit masks lm[li] & RT[b'] (row-independent) computed once; row x's
// hits of item k are that mask & the row's slot mask.  Row x's arcs of word w start at arcbase[block] +
// warc[word] (k_tile_count, k_block_counts).  Per (row, word): walk 1 -- the per-state arc counts and
// a warp scan give each state's first arc slot; walk 2 writes the arc codes in (state, item, slot)
// order; then lanes take CONSECUTIVE arcs (coalesced streaming stores of dst / ilabel / olabel /
// weight).
template <int kJ>
__global__ void __launch_bounds__(kEThreads, 1) k_tile_emit(Ctx cx, TileArgs ta, EmitIO io,
                                                             const int64_t* __restrict__ tot, int vr_rows) {
  __shared__ TileSmem<uint32_t> t;
  __shared__ int32_t rbase[kESlots];
  extern __shared__ __align__(16) uint32_t tdyn[];
  const TC c = tc_of(cx);
  const int wpr = c.wpr, VB = c.VB, bpr = c.bpr, wd = ta.sd.wd;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* RT = tdyn;                                                  // [wpr * 32]
  uint32_t* Vw = RT + (size_t)wpr * 32;                                 // [vr_rows * wpr]
  uint16_t* Pw = (uint16_t*)(Vw + (size_t)vr_rows * wpr);                // [vr_rows * wpr]
  uint32_t* code = Vw + (size_t)vr_rows * wpr + ((size_t)vr_rows * wpr + 1) / 2 + (size_t)warp * kECap;
  const int64_t id_comp = tot[0], arc_comp = tot[1];
  const uint32_t* __restrict__ V = cx.V;
  for (int tile = ta.t0 + blockIdx.x; tile < ta.t1; tile += gridDim.x) {
    tile_slots(t, ta, tile);
    const int nr = t.nr, ns = t.ns;
    const int32_t r0 = t.r0;
    for (int k = warp; k < ns; k += kEWarps) {  // stage the slot rows: a warp per row, coalesced
      const int32_t row = t.srow[k];
      const int64_t gw0 = c.W + (int64_t)row * wpr, kb = c.K + (int64_t)row * bpr;
      const int64_t ib = __ldg(&cx.idbase[kb]);
      if (lane == 0) rbase[k] = (int32_t)(ib - id_comp);
      for (int w0 = lane; w0 < wpr; w0 += 4 * 32) {
        uint32_t v[4], pr[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int w = w0 + 32 * u;
          v[u] = pr[u] = 0u;
          if (w < wpr) {
            v[u] = __ldg(&V[gw0 + w]);
            pr[u] = (uint32_t)(__ldg(&cx.idbase[kb + (w >> 5)]) - ib + __ldg(&cx.wpre[gw0 + w]));
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int w = w0 + 32 * u;
          if (w < wpr) {
            Vw[(size_t)k * wpr + w] = v[u];
            Pw[(size_t)k * wpr + w] = (uint16_t)pr[u];
          }
        }
      }
    }
    __syncthreads();
    // RT from the staged slot rows (lane s reads row s: bank (s * wpr + w) % 32, conflict-free for odd wpr)
    for (int w = warp; w < wpr; w += kEWarps) {
      const uint32_t x = lane < ns ? Vw[lane * wpr + w] : 0u;
      RT[w * 32 + lane] = transpose32(x, lane);
    }
    __syncthreads();
    const int j0 = t.lm[kLiSent] ? 0 : 1;
    const uint32_t selfm = t.selfm;
    const uint32_t* lm = t.lm;
    // lane x < nr: row x's slot mask and start / accept flags (bits 0 / 1)
    const uint32_t rm_l = lane < nr ? t.rmask[lane] : 0u;
    const uint32_t fl_l = lane < nr ? (uint32_t)__ldg(&io.startA[r0 + lane]) | ((uint32_t)__ldg(&io.accA[r0 + lane]) << 1) : 0u;
    for (int w = warp; w < wpr; w += kEWarps) {
      // lane x < nr: V word of (row x, w), the id of its first state, the arc base and arc count
      uint32_t vw_l = 0u;
      int32_t id_l = 0, exp_l = 0;
      int64_t base_l = 0;
      if (lane < nr && c.own(r0 + lane)) {  // (rows of other shards are emitted there)
        const int64_t gw = c.W + (int64_t)(r0 + lane) * wpr + w;
        const int64_t blk = c.K + (int64_t)(r0 + lane) * bpr + (w >> 5);
        vw_l = __ldg(&V[gw]);
        id_l = (int32_t)(__ldg(&cx.idbase[blk]) - id_comp + __ldg(&cx.wpre[gw]));
        const uint32_t pre = __ldg(&cx.warc[gw]);
        base_l = __ldg(&cx.arcbase[blk]) - arc_comp + pre;
        const bool last = (w & 31) == 31 || w == wpr - 1;
        exp_l = (int32_t)((last ? (uint32_t)__ldg(&cx.kept[blk]) : __ldg(&cx.warc[gw + 1])) - pre);
      }
      if (!__any_sync(0xffffffffu, vw_l != 0u)) continue;
      const int b = w * 32 + lane;
      const bool inb = b < VB;
      const int jn = ta.sd.wmax[w];
      const uint32_t* __restrict__ ellw = ta.sd.ell + (size_t)w * wd * 32 + lane;
      const int2* __restrict__ cww = ta.sd.ellcw + (size_t)w * wd * 32;
      // per item: hit slots of all tile rows (g) and the code's item bits (cb)
      uint32_t g[kJ + 1], cb[kJ + 1];
#pragma unroll
      for (int k = 0; k <= kJ; ++k) {
        const uint32_t xi = (inb && (k == 0 ? j0 == 0 : k < jn)) ? __ldg(ellw + k * 32) : (kLiPad << 24);
        g[k] = lm[xi >> 24] & RT[xi & 0xFFFFFFu];
        cb[k] = ((xi & 0xFFFFu) << 15) | ((uint32_t)k << 10) | ((uint32_t)lane << 5);
      }
      for (int x = 0; x < nr; ++x) {
        const uint32_t vw = __shfl_sync(0xffffffffu, vw_l, x);
        if (!vw) continue;
        const int64_t run = __shfl_sync(0xffffffffu, base_l, x);
        const uint32_t rmx = __shfl_sync(0xffffffffu, rm_l, x);
        const uint32_t rmv = ((vw >> lane) & 1u) ? rmx : 0u;
        // walk 1: the state's arc count
        int cnt = 0;
#pragma unroll
        for (int k = 0; k <= kJ; ++k) cnt += __popc(g[k] & rmv);
        for (int j = kJ + 1; j < jn; ++j) {  // (wide B rows: items beyond the registers)
          const uint32_t xi = inb ? __ldg(ellw + j * 32) : (kLiPad << 24);
          cnt += __popc(lm[xi >> 24] & RT[xi & 0xFFFFFFu] & rmv);
        }
        const int inc = warp_incl_scan(cnt);
        const int ex = inc - cnt;
        const int T = __shfl_sync(0xffffffffu, inc, 31);
        if (lane == x && T != exp_l) atomicAdd(&cx.misc[2], 1ull);
        {
          const int32_t idw = __shfl_sync(0xffffffffu, id_l, x);
          const uint32_t fl = __shfl_sync(0xffffffffu, fl_l, x);
          if (rmv) {  // the state's own outputs
            const int32_t id = idw + __popc(vw & ((1u << lane) - 1u));
            __stcs((long long*)&io.row_ptr[id], (long long)(run + ex));
            __stcs(&io.pair_a[id], r0 + x);
            __stcs(&io.pair_b[id], b);
            io.is_start[id] = (uint8_t)((fl & 1u) & __ldg(&io.startB[b]));
            io.is_accept[id] = (uint8_t)((fl >> 1) & __ldg(&io.accB[b]));
          }
        }
        // phase 3: arcs [p, p + n) of the (row, word) from the code buffer
        auto flush = [&](int p, int n) {
          __syncwarp();
          for (int i0 = lane; i0 < n; i0 += 64) {  // two arcs per lane in flight
            int2 cw[2];
            uint32_t cd[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int i = i0 + 32 * u;
              cd[u] = i < n ? code[i] : 0u;
              cw[u] = (i < n && (cd[u] & (31u << 10))) ? __ldg(cww + ((cd[u] >> 5) & 1023u)) : make_int2(0, 0);
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int i = i0 + 32 * u;
              if (i >= n) break;
              const uint32_t o = cd[u] >> 15;
              const int s = cd[u] & 31;
              const uint32_t vword = Vw[s * wpr + (o >> 5)];
              const int32_t did = rbase[s] + Pw[s * wpr + (o >> 5)] + __popc(vword & ((1u << (o & 31)) - 1u));
              int32_t il, ol;
              float wt;
              if (!(cd[u] & (31u << 10))) {  // item 0 = M2: A eps arc, B stays (bit copy)
                il = t.scarry[s];
                ol = FST_EPS;
                wt = t.sw[s];
              } else if ((selfm >> s) & 1u) {  // M3: B eps arc, A stays (bit copy)
                il = FST_EPS;
                ol = cw[u].x;
                wt = __int_as_float(cw[u].y);
              } else {                         // M1: one binary32 add, RN-even
                il = t.scarry[s];
                ol = cw[u].x;
                wt = __fadd_rn(t.sw[s], __int_as_float(cw[u].y));
              }
              const int64_t q = run + p + i;
              __stcs(&io.dst[q], did);
              __stcs(&io.ilabel[q], il);
              __stcs(&io.olabel[q], ol);
              __stcs(&io.weight[q], wt);
            }
          }
          __syncwarp();
        };
        if (T <= kECap) {  // walk 2, one flush (the common case: no range tests)
          uint32_t* cp = code + ex;
#pragma unroll
          for (int k = 0; k <= kJ; ++k) {
            uint32_t hj = g[k] & rmv;
            while (hj) {
              *cp++ = cb[k] | (uint32_t)(__ffs(hj) - 1);
              hj &= hj - 1u;
            }
          }
          for (int j = kJ + 1; j < jn; ++j) {
            const uint32_t xi = inb ? __ldg(ellw + j * 32) : (kLiPad << 24);
            uint32_t hj = lm[xi >> 24] & RT[xi & 0xFFFFFFu] & rmv;
            const uint32_t cj = ((xi & 0xFFFFu) << 15) | ((uint32_t)j << 10) | ((uint32_t)lane << 5);
            while (hj) {
              *cp++ = cj | (uint32_t)(__ffs(hj) - 1);
              hj &= hj - 1u;
            }
          }
          flush(0, T);
          continue;
        }
        for (int p = 0; p < T; p += kECap) {
          // walk 2: arc codes of positions [p, p + kECap)
          if (cnt && ex < p + kECap && ex + cnt > p) {
            int pos = ex;
            auto put = [&](uint32_t hj, uint32_t hi) {
              while (hj) {
                const int s = __ffs(hj) - 1;
                hj &= hj - 1u;
                if (pos >= p && pos < p + kECap) code[pos - p] = hi | s;
                ++pos;
              }
            };
#pragma unroll
            for (int k = 0; k <= kJ; ++k) put(g[k] & rmv, cb[k]);
            for (int j = kJ + 1; j < jn; ++j) {
              const uint32_t xi = inb ? __ldg(ellw + j * 32) : (kLiPad << 24);
              put(lm[xi >> 24] & RT[xi & 0xFFFFFFu] & rmv, ((xi & 0xFFFFu) << 15) | ((uint32_t)j << 10) | ((uint32_t)lane << 5));
            }
          }
          flush(p, min(kECap, T - p));
        }
      }
    }
    __syncthreads();
  }
}

// B-role ELL of a view, word-tiled: item j of node b at [(b / 32) * wd + j][b % 32]; column 0 = the
// sentinel item (b itself), columns 1.. = the node's arcs in view order, padded; wmax[word] = columns
// used by the word's 32 nodes; *has_eps |= any eps key.
__global__ void k_build_ell(int32_t V, const int32_t* __restrict__ off, const int32_t* __restrict__ key,
                            const int32_t* __restrict__ other, const int2* __restrict__ cw, int wd, uint32_t* ell,
                            int2* ellcw, uint8_t* wmax, int32_t* has_eps) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  int d = 0;
  bool eps = false;
  const size_t base = (size_t)(b >> 5) * wd * 32 + lane;
  if (b < V) {
    const int32_t e0 = off[b];
    d = off[b + 1] - e0;
    ell[base] = (kLiSent << 24) | (uint32_t)b;
    if (ellcw) ellcw[base] = make_int2(0, 0);
    for (int j = 1; j < wd; ++j) {
      const int k = j - 1;
      if (k < d) {
        const int32_t l = key[e0 + k];
        eps |= l == FST_EPS;
        ell[base + (size_t)j * 32] = ((uint32_t)(l + 2) << 24) | (uint32_t)other[e0 + k];
        if (ellcw) ellcw[base + (size_t)j * 32] = cw[e0 + k];
      } else {
        ell[base + (size_t)j * 32] = kLiPad << 24;
        if (ellcw) ellcw[base + (size_t)j * 32] = make_int2(0, 0);
      }
    }
  } else if ((b >> 5) * 32 < V) {  // padding lanes of the last word
    for (int j = 0; j < wd; ++j) {
      ell[base + (size_t)j * 32] = kLiPad << 24;
      if (ellcw) ellcw[base + (size_t)j * 32] = make_int2(0, 0);
    }
  }
  const unsigned m = __reduce_max_sync(0xffffffffu, (unsigned)(b < V ? d + 1 : 0));
  if (lane == 0 && b < V) wmax[b >> 5] = (uint8_t)m;
  if (__any_sync(0xffffffffu, eps) && lane == 0) atomicOr(has_eps, 1);
}
