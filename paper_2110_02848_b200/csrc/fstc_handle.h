// fstc_handle.h -- host-side definition of the opaque fst handle.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <vector>

#include "../../include/fstc.h"

namespace fstc {

void release_buffer(void* ptr, size_t bytes, cudaStream_t s);  // memory.cu

// Stream-ordered device allocation, released on the owning stream (large buffers go back to the
// library's buffer cache, see memory.cu).
struct DeviceBuffer {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaStream_t stream = nullptr;
  ~DeviceBuffer() {
    if (ptr) release_buffer(ptr, bytes, stream);
  }
};
using BufferPtr = std::shared_ptr<DeviceBuffer>;

// Allocates `bytes` (rounded up to 256 B) on `s`'s pool; returns nullptr-holding ptr on failure.
fst_status alloc_buffer(size_t bytes, cudaStream_t s, BufferPtr* out);

enum ViewId { kOutByOlabel = 0, kInByOlabel = 1, kOutByIlabel = 2, kInByIlabel = 3 };

struct View {
  int32_t* off = nullptr;    // [V+1]
  int32_t* key = nullptr;    // [E]
  int32_t* other = nullptr;  // [E]
  int32_t* carry = nullptr;  // [E]
  float* w = nullptr;        // [E]
  int32_t* arc = nullptr;    // [E] original arc index
  int2* cw = nullptr;        // [E] packed (carry, weight bits): the per-arc data of the emit
  int2* ikd = nullptr;       // [E+V] items: per node a sentinel (kSentinel, node) then (key, other) of its arcs
  int32_t* isrc = nullptr;   // [E+V] item -> node
  int4* ikcw = nullptr;      // [E+V] items with (key, other, carry, weight bits); sentinel = (kSentinel, node, 0, 0)
  // label-major segment index (B-role views): arcs ordered by (label, node, view position); a
  // segment is a run of equal (label, node)
  int32_t* lm_other = nullptr;  // [E] other-end node
  int32_t* lm_pos = nullptr;    // [E] view position
  int32_t* seg_node = nullptr;  // [E] node of segment s
  int32_t* seg_beg = nullptr;   // [E+1] first label-major index of segment s
  int32_t* lab_val = nullptr;   // [E] distinct labels, ascending
  int32_t* lab_seg = nullptr;   // [E+1] first segment of each distinct label
  int32_t nseg = 0, nlab = 0;
  int32_t max_deg = 0;  // largest node degree of the view
};

}  // namespace fstc

struct fst {
  bool composed = false;
  int32_t V = 0;
  int64_t E = 0;
  cudaStream_t stream = nullptr;
  // the CSR (device)
  int64_t* row_ptr = nullptr;
  int32_t* ilabel = nullptr;
  int32_t* olabel = nullptr;
  int32_t* dst = nullptr;
  float* weight = nullptr;
  uint8_t* is_start = nullptr;
  uint8_t* is_accept = nullptr;
  int32_t* pair_a = nullptr;
  int32_t* pair_b = nullptr;
  int32_t* arc_a = nullptr;  // provenance (composed with FST_COMPOSE_PROVENANCE)
  int32_t* arc_b = nullptr;
  int32_t* pair_f = nullptr;  // eps-filter state of every state (FST_COMPOSE_EPS_FILTER), else nullptr
  bool filtered = false;
  int64_t src_arcs_a = 0, src_arcs_b = 0;  // arc counts of the inputs (grad_a / grad_b lengths)
  // label-sorted views (built by fst_create, lazily for composed handles)
  bool has_views = false;
  fstc::View views[4];
  int32_t* start_list = nullptr;
  int32_t* accept_list = nullptr;
  int32_t n_start = 0, n_accept = 0;
  int32_t max_ilabel = -1, max_olabel = -1;
  fst_compose_stats stats{};
  // sharded compositions: this handle holds rank `shard_rank`'s rows (global state ids in dst)
  int32_t shard_rank = -1, shard_world = 0;
  int64_t shard_state_offset = 0, shard_arc_offset = 0, shard_total_states = 0, shard_total_arcs = 0;
  std::vector<int64_t> level_sizes[2];  // frontier size per BFS level, stage 1 / stage 2
  std::vector<fstc::BufferPtr> buffers;  // owned (or shared with a batch) device memory
  std::vector<cudaEvent_t> use_events;   // async work on other streams that reads the buffers (fst_free waits)
  // tile path caches (compose.cu / tile.cuh), built on first use; a handle is immutable
  struct TileEll {  // B role: ELL of a view ([0] out-by-ilabel with (carry, weight), [1] in-by-ilabel)
    bool ok = false;
    fstc::BufferPtr buf;
    uint32_t* ell = nullptr;
    int2* cw = nullptr;
    uint8_t* wmax = nullptr;
    int32_t wd = 0;
    bool has_eps = false;
  } tile_ell[2];
  struct TileRows {  // A role: tile row starts for (view, self slot, caps)
    int64_t key = 0;
    fstc::BufferPtr buf;
    int32_t* d = nullptr;
    int32_t n = 0;
    std::vector<int32_t> h;  // host copy (the sharded path picks each rank's tiles)
  };
  std::vector<TileRows> tile_rows;
  std::vector<int32_t> tile_hoff[2];  // host copy of the A-role view offsets ([0] out, [1] in by olabel)
  // wave path caches (wave.cu), built on first use
  int8_t a_topo = -1;  // A role: 1 if every arc has src < dst (rows in topological order), 0 if not
  struct WaveEll {     // B role, [0] out-by-ilabel, [1] in-by-ilabel: ELL of the light columns by word
    bool ok = false;
    fstc::BufferPtr buf;
    uint32_t* ell = nullptr;   // non-eps items: [(woff[w] + j) * 32 + lane] = (label + 2) << 24 | other; 255 << 24 = pad
    uint32_t* woff = nullptr;  // [wpr + 1] first ELL row of each word
    uint8_t* wmax = nullptr;   // [wpr] ELL rows of each word (max light non-eps degree in the word)
    uint32_t* eell = nullptr;  // eps items of the light columns, same layout
    uint32_t* ewoff = nullptr;
    uint8_t* ewmax = nullptr;
    uint32_t blab[8] = {};     // label indices (label + 2) of the light non-eps items
    int2* ellcw = nullptr;     // [0] only: (olabel, weight bits) parallel to ell / eell / hitems (the emit)
    int2* eellcw = nullptr;
    int2* hcw = nullptr;
    uint32_t* hbefore = nullptr;  // [wpr + 1] heavy columns before each word
    uint32_t* wo = nullptr;       // [wpr + 1] woff << 8 | wmax
    uint32_t* ewo = nullptr;      // [wpr + 1] ewoff << 8 | ewmax
    uint32_t* hmask = nullptr; // [wpr] lanes of heavy columns
    int4* heavy = nullptr;     // (col, first item, first non-eps item, end) of heavy columns, by col
    int32_t nheavy = 0;
    int2* eps = nullptr;       // [0] only: B arcs with ilabel eps as (src, dst), dst not a hub
    int32_t neps = 0;
    int32_t nhub = 0;          // [0] only: eps hub targets (many eps in-arcs)
    int32_t* hub_col = nullptr;
    uint32_t* hub_src = nullptr;  // [nhub][wpr] eps sources of each hub
    uint32_t* hitems = nullptr;   // items of the heavy columns, packed like the ELL
    uint32_t* rel = nullptr;      // [0] only: [4][wpr] relevance masks of the M3 passes (wave.cu)
  } wave_ell[2];
};
