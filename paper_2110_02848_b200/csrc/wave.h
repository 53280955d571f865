// wave.h -- the wave path (wave.cu): row-by-row stages for compositions whose A is
// topologically numbered.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fstc.h"

namespace fstc {

struct WavePlan {
  bool ok = false;
  int32_t depth = 0;    // row steps of the longest composition (sequential per cluster)
  int32_t cluster = 1;  // CTAs per cluster (one composition per cluster)
  bool emit_ok = false;  // the wave emit's staged rows fit in shared memory (else the general emit runs)
  struct Impl;
  Impl* impl;
  WavePlan();
  ~WavePlan();
  WavePlan(const WavePlan&) = delete;
  WavePlan& operator=(const WavePlan&) = delete;
};

// plan->ok when every composition qualifies (A topologically numbered, A rows <= 64 arcs, B ilabels
// <= 252, V_B < 2^24; automatic mode: V_A <= 4096) and the wave mode allows it.  W / K: first word /
// block of each composition's pair space.
fst_status wave_plan(int32_t n, const fst_handle* a, const fst_handle* b, const int64_t* W, const int64_t* K,
                     cudaStream_t s, WavePlan* plan);
// stage 1 writes every word of R, stage 2 every word of V (reads R).
fst_status wave_stage(const WavePlan& plan, int stage, uint32_t* R, uint32_t* V, cudaStream_t s);
// pass-1 counts of every pair of R (cnt8, saturated; exact for heavy states): needs only R, so it may run
// on another stream concurrently with stage 2.
fst_status wave_count(const WavePlan& plan, uint32_t* R, uint8_t* cnt8, cudaStream_t s);
// pass-1 block sums over V: kept[] of every block (overwritten); after wave_count and stage 2.
fst_status wave_kept(const WavePlan& plan, uint32_t* V, unsigned long long* kept, cudaStream_t s);
// pass 2 (general emit replacement; no provenance; needs plan.emit_ok): writes every composition's CSR from the numbering
// (idbase / arcbase per block, wpre per word).  `err` counts internal inconsistencies (must stay 0).
fst_status wave_emit(const WavePlan& plan, const struct CompDev* d_comps, const int64_t* d_tot, const int64_t* idbase,
                     const int64_t* arcbase, const uint16_t* wpre, uint32_t* V, int32_t* err, cudaStream_t s);
void wave_mode_set(int mode);

}  // namespace fstc
