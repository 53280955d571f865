// fstc_internal.cuh -- internal data structures of libfstc (B200 / sm_100a).
//
// Layout in HBM:
//   * Input FST handle: the CSR as given plus four label-sorted adjacency VIEWS (SoA, int32):
//       out-by-olabel (A role, forward), in-by-olabel (A role, backward),
//       out-by-ilabel (B role, forward), in-by-ilabel (B role, backward).
//     Each view: off[V+1], key[E] (the matched label, ascending within a node, eps = -1 first so
//     eps arcs are a prefix), other[E] (dst for out-views, src for in-views), carry[E] (the label
//     that is copied to the output: ilabel for the A role, olabel for the B role), w[E], arc[E].
//   * Pair space of a composition: V_A rows of ceil(V_B/32) 32-bit words; bit (a,b) lives in word
//     W + a*wpr + b/32, bit b%32.  Rows are split into BLOCKS of 32 words (1024 pairs), the unit of
//     frontier scheduling and of state / arc numbering.  Batches concatenate pair spaces
//     (W, K = word / block bases per composition).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fstc.h"

namespace fstc {

constexpr int kWordsPerBlock = 32;    // 32 words x 32 bits = 1024 pairs per block
constexpr int kPairsPerBlock = 1024;

struct ViewDev {
  const int32_t* off;    // [V+1]
  const int32_t* key;    // [E] matched label, sorted within node
  const int32_t* other;  // [E] other-end node
  const int32_t* carry;  // [E] label carried to the output
  const float* w;        // [E] weight
  const int2* cw;         // [E] packed (carry, weight bits)
  const int2* ikd;        // [E+V] items: node v owns items [off[v]+v, off[v+1]+v+1): a sentinel
                          //       (kSentinel, v) then (key, other) of its arcs in view order
  const int32_t* isrc;    // [E+V] item -> node
  const int4* ikcw;       // [E+V] items with (key, other, carry, weight bits)
  // label-major segment index (B role): see View in fstc_handle.h
  const int32_t* lm_other;
  const int32_t* lm_pos;
  const int32_t* seg_node;
  const int32_t* seg_beg;
  const int32_t* lab_val;
  const int32_t* lab_seg;
  int32_t nlab;
  const int32_t* arc;     // [E] view position -> input arc index (provenance)
};

constexpr int32_t kSentinel = INT32_MIN;

// One composition inside a (possibly batched) call.
struct CompDev {
  ViewDev Af, Ab, Bf, Bb;  // forward (out) / backward (in) views of A (by olabel) and B (by ilabel)
  const uint8_t* startA;
  const uint8_t* startB;
  const uint8_t* accA;
  const uint8_t* accB;
  const int32_t* startListA;
  const int32_t* startListB;
  const int32_t* accListA;
  const int32_t* accListB;
  int32_t nStartA, nStartB, nAccA, nAccB;
  int32_t VA, VB;
  int32_t wpr, bpr;  // words per row, blocks per row
  int32_t cpr, CB;   // chunks per row, blocks per chunk (a chunk is one CTA task)
  int32_t smallA;    // A's olabels < 63: label-mask matching of an A row is possible
  int64_t W;         // first word of this composition's pair space
  int64_t K;         // first block
  int64_t Q;         // first chunk
  int32_t sh_world, sh_rank;  // sharded composition (world > 1): see owned() / blk_owner()
  int32_t sh_rows;            // 1: rank q owns the rows [V_A*q/world, V_A*(q+1)/world); 0: block-interleaved
  int32_t sh_r0, sh_r1;       // rows mode: this rank's rows
  // outputs (filled before the emit kernel; for a shard they are biased so that a global state id /
  // arc slot indexes the shard's own buffers)
  int64_t* row_ptr;
  int32_t* ilabel;
  int32_t* olabel;
  int32_t* dst;
  float* weight;
  uint8_t* is_start;
  uint8_t* is_accept;
  int32_t* pair_a;
  int32_t* pair_b;
  int32_t* arc_a;  // provenance outputs (FST_COMPOSE_PROVENANCE), nullptr when off
  int32_t* arc_b;
};

// Per-level control block (ring of 3).
struct LevelCtrl {
  unsigned long long count;    // number of active chunks in the list of this level
  unsigned long long nnew;     // states discovered (claimed) into this level's frontier
  unsigned long long pad[2];
};

constexpr int kMaxLevelStats = 1 << 16;

// Ownership of pair-space blocks in a sharded composition.  Block-interleaved mode: the
// 1024-pair block j of row a has linear id a * bpr + j and belongs to rank (id mod world) -- every row
// is spread over all ranks (trellis-shaped compositions).  Rows mode (compositions on the tile path):
// rank q owns the contiguous rows [V_A*q/world, V_A*(q+1)/world), so its tiles are its own.
__device__ __host__ __forceinline__ int32_t sh_row0(const CompDev& C, int q) {
  return (int32_t)(((int64_t)C.VA * q) / C.sh_world);
}
__device__ __forceinline__ int blk_owner(const CompDev& C, int64_t blk) {
  if (C.sh_world <= 1) return 0;
  if (!C.sh_rows) return (int)(blk % C.sh_world);
  const int32_t row = (int32_t)(blk / C.bpr);
  int q = (int)(((int64_t)row * C.sh_world) / (C.VA > 0 ? C.VA : 1));
  while (q + 1 < C.sh_world && sh_row0(C, q + 1) <= row) ++q;
  while (q > 0 && sh_row0(C, q) > row) --q;
  return q;
}
__device__ __forceinline__ bool owned(const CompDev& C, int32_t row, int32_t col) {
  if (C.sh_world <= 1) return true;
  if (C.sh_rows) return row >= C.sh_r0 && row < C.sh_r1;
  return (((int64_t)row * C.bpr + (col >> 10)) % C.sh_world) == C.sh_rank;
}
// Blocks of rank q in block-id order: the p-th is owner_block(C, q, p); owner_nblocks(C, q) of them.
__device__ __host__ __forceinline__ int64_t owner_nblocks(const CompDev& C, int q) {
  const int64_t nb = (int64_t)C.VA * C.bpr;
  if (C.sh_world <= 1) return nb;
  if (C.sh_rows) return (int64_t)(sh_row0(C, q + 1) - sh_row0(C, q)) * C.bpr;
  return nb > q ? (nb - q + C.sh_world - 1) / C.sh_world : 0;
}
__device__ __host__ __forceinline__ int64_t owner_block(const CompDev& C, int q, int64_t p) {
  if (C.sh_world <= 1) return p;
  if (C.sh_rows) return (int64_t)sh_row0(C, q) * C.bpr + p;
  return p * C.sh_world + q;
}

__device__ __forceinline__ int find_comp(const CompDev* __restrict__ comps, int ncomp, int64_t blk) {
  // largest i with comps[i].K <= blk
  int lo = 0, hi = ncomp - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (comps[mid].K <= blk) lo = mid; else hi = mid - 1;
  }
  return lo;
}

}  // namespace fstc

// ---------------------------------------------------------------------------------------------
// host-side helpers shared by the translation units
namespace fstc {
void set_error(fst_status st, const char* fmt, ...);
void count_launch(int64_t n = 1);
int sm_count();
}  // namespace fstc

#define FSTC_CUDA_TRY(expr)                                                                   \
  do {                                                                                        \
    cudaError_t _e = (expr);                                                                  \
    if (_e != cudaSuccess) {                                                                  \
      fstc::set_error(FST_E_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),     \
                      __FILE__, __LINE__);                                                    \
      return _e == cudaErrorMemoryAllocation ? FST_E_OOM : FST_E_CUDA;                        \
    }                                                                                         \
  } while (0)

#define FSTC_LAUNCH_CHECK()                                                                   \
  do {                                                                                        \
    fstc::count_launch();                                                                     \
    cudaError_t _e = cudaGetLastError();                                                      \
    if (_e != cudaSuccess) {                                                                  \
      fstc::set_error(FST_E_CUDA, "kernel launch failed: %s (%s:%d)", cudaGetErrorString(_e), \
                      __FILE__, __LINE__);                                                    \
      return FST_E_CUDA;                                                                      \
    }                                                                                         \
  } while (0)
