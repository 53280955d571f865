/*
 * fstc.h -- C ABI of the B200-native eager WFST composition library (libfstc.so).
 *
 * The library implements the data-parallel hot path of arXiv 2110.02848 ("parallel composition
 * of WFSTs on GPUs"): eager, trimmed composition C = A o B in the log semiring with epsilon
 * transitions.  The calls follow the paper's statement of the problem -- "Input: Transducers A and
 * B ... Return: The composed graph C" (Algorithm 1) -- over the
 * structure-of-arrays transducer of §3.2 (start/accept flags, per-arc label /
 * weight / node arrays, per-node arc offsets).
 *
 * Semantics:
 *   * epsilon = FST_EPS (-1).  Labels are int32 >= -1.  Only A.olabel and B.ilabel are matched.
 *   * Moves from a pair (u_a,u_b) -- reading N1:
 *       M1  e_a in out(u_a), e_b in out(u_b), olabel(e_a) == ilabel(e_b) (eps == eps included)
 *           -> (dst e_a, dst e_b), label ilabel(e_a):olabel(e_b), weight fl32(w_a + w_b)
 *       M2  e_a with olabel eps, B stays -> (dst e_a, u_b), label ilabel(e_a):eps, weight w_a (bits)
 *       M3  e_b with ilabel eps, A stays -> (u_a, dst e_b), label eps:olabel(e_b), weight w_b (bits)
 *   * Output = trim(product): exactly the pairs reachable from a start pair (S_A x S_B) AND
 *     co-accessible to an accept pair (F_A x F_B), with every move between them.
 *   * Output numbering: states in ascending pair key  a * V_B + b ; arcs of a state in a fixed
 *     deterministic enumeration order.  Repeated calls give bit-identical outputs.
 *
 * Threading / streams: every call takes a CUDA stream (cudaStream_t passed as void*; NULL = the
 * legacy default stream).  fst_create and fst_compose* are BLOCKING: they return when their
 * results are complete (composition sizes are data dependent).  Handles are immutable after
 * creation and may be shared by concurrent calls on different streams.
 *
 * Errors: every fst_status != FST_OK leaves the outputs untouched (or NULL) and sets a
 * thread-local message readable with fst_last_error().  There is no CPU fallback: if no CUDA
 * device is usable the calls fail with FST_E_CUDA.
 */
#ifndef FSTC_H_
#define FSTC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FST_EPS (-1) /* epsilon label (reading 1) */

typedef struct fst* fst_handle; /* opaque; owns its device memory */

typedef enum {
  FST_OK = 0,
  FST_E_INVALID_ARG = 1,   /* NULL pointer, negative size, n < 0, ... */
  FST_E_INVALID_GRAPH = 2, /* fst_create validation failed (see fst_desc) */
  FST_E_OOM = 3,           /* device allocation failed */
  FST_E_CAPACITY = 4,      /* pair space / output beyond what the library can address */
  FST_E_CUDA = 5,          /* CUDA runtime error (message in fst_last_error) */
  FST_E_NCCL = 6,          /* reserved for the sharded multi-GPU mode */
  FST_E_INTERNAL = 7       /* internal consistency check failed (a bug) */
} fst_status;

typedef enum { FST_MEM_DEVICE = 0, FST_MEM_HOST = 1 } fst_memory;

/* Input transducer, CSR grouped by source state ("five arrays each with E
 * entries" + "outArcOffset").  Arcs of state v are [row_ptr[v], row_ptr[v+1]); their order inside a
 * row is arbitrary (the library builds its own label-sorted views).  All arrays are BORROWED for
 * the duration of fst_create only and live in device memory (memory = FST_MEM_DEVICE) or in host
 * memory (FST_MEM_HOST; pinned memory gives the fastest upload).  Validated, else
 * FST_E_INVALID_GRAPH: row_ptr[0] == 0, non-decreasing, row_ptr[V] == E; 0 <= dst < V;
 * labels >= -1; weights finite (no NaN / +-inf); flags in {0,1}.  V < 2^31, E < 2^31. */
typedef struct {
  int32_t num_states;       /* V >= 0 */
  int64_t num_arcs;         /* E >= 0 */
  const int64_t* row_ptr;   /* [V+1] */
  const int32_t* ilabel;    /* [E] input label  */
  const int32_t* olabel;    /* [E] output label */
  const int32_t* dst;       /* [E] destination state ("output node") */
  const float* weight;      /* [E] log-semiring weight */
  const uint8_t* is_start;  /* [V] start flags */
  const uint8_t* is_accept; /* [V] accept flags */
  int32_t memory;           /* fst_memory: where the arrays above live */
} fst_desc;

/* Read-only view of a handle's arrays (DEVICE pointers owned by the handle, valid until fst_free).
 * Composed graphs also carry pair_a/pair_b: the (a,b) pair of every state (SPEC "pairKeys");
 * they are NULL for handles made by fst_create. */
typedef struct {
  int32_t num_states;
  int64_t num_arcs;
  const int64_t* row_ptr; /* [V+1] */
  const int32_t* ilabel;  /* [E] */
  const int32_t* olabel;  /* [E] */
  const int32_t* dst;     /* [E] */
  const float* weight;    /* [E] */
  const uint8_t* is_start;
  const uint8_t* is_accept;
  const int32_t* pair_a; /* [V] or NULL */
  const int32_t* pair_b; /* [V] or NULL */
  const int32_t* arc_a;  /* [E] provenance (FST_COMPOSE_PROVENANCE), else NULL: see fst_compose_ex */
  const int32_t* arc_b;  /* [E] */
  const int32_t* pair_f; /* [V] eps-filter state f of every state (FST_COMPOSE_EPS_FILTER), else NULL */
} fst_view;

/* Per-composition statistics (filled by fst_compose*; timings only when profiling is on). */
typedef struct {
  int32_t levels_stage1;  /* BFS levels of the backward co-accessibility stage (Alg. 1 line 3) */
  int32_t levels_stage2;  /* BFS levels of the forward stage (Alg. 1 lines 12-31) */
  int64_t num_coaccessible; /* |R| over the pair space (profiling only; else -1) */
  int64_t pair_space;     /* V_A * V_B summed over the call */
  float ms_stage1;        /* CUDA-event time of the backward BFS (profiling only) */
  float ms_stage2;        /* forward BFS */
  float ms_number;        /* popcount directory + scans (+ |R| when profiling) */
  float ms_alloc;         /* output allocation */
  float ms_emit;          /* emit kernel (writes the composed CSR) */
  float ms_total;         /* whole call */
  int64_t launches;       /* kernels launched by the call */
  int64_t emit_launches;  /* of which emit kernels */
  int64_t expand_launches;/* of which BFS level kernels */
  int64_t staged_tasks;   /* chunk tasks of the BFS levels that used shared-memory staging (wave path: CTAs per cluster) */
  int32_t tile_path;      /* 1: the call ran the tile kernels (bottom-up levels, count, emit);
                             2: the wave kernels (row-by-row stages for a topologically numbered A, §6c) */
  int32_t pull_levels;    /* BFS rounds (both stages) that ran bottom-up on the tile kernels */
  float ms_count;         /* tile path: pass-1 count kernel (profiling only; included in ms_stage2); wave path:
                             the counts on the side stream, concurrent with stage 2 (not additive) */
} fst_compose_stats;

/* Upload + validate + build label-sorted adjacency views.  On success *out is a
 * new handle.  Synchronises `stream`. */
fst_status fst_create(const fst_desc* desc, void* stream, fst_handle* out);

/* C = trim(A o B) (Algorithm 1 semantics, two-stage frontier BFS on the GPU).  *c receives a new
 * handle (possibly with 0 states: an empty result is FST_OK).  a and b may be the same handle. */
fst_status fst_compose(fst_handle a, fst_handle b, void* stream, fst_handle* c);

/* n independent compositions c[i] = a[i] o b[i] advanced together in one level loop over
 * concatenated pair spaces.  All-or-nothing: on error every c[i] is NULL. */
fst_status fst_compose_batch(int32_t n, const fst_handle* a, const fst_handle* b, void* stream,
                             fst_handle* c);

/* Option flags of fst_compose_ex / fst_compose_batch_ex. */
#define FST_COMPOSE_PROVENANCE 1u /* also record, per composed arc, the arc pair that produced it */
#define FST_COMPOSE_EPS_FILTER 2u /* three-state eps filter: no duplicated eps paths (see below) */

/* fst_compose / fst_compose_batch with option flags.  FST_COMPOSE_PROVENANCE (
 * the autodiff use of the composed graph): every arc k of C also gets
 * arc_a[k] = the index of the A arc e_a of its move in A's input arc order (the order of the
 * fst_desc passed to fst_create; for a composed A, its own arc order), or -1 for an M3 move
 * (A stays), and arc_b[k] = the B arc e_b, or -1 for an M2 move (B stays) -- Alg. 1 line 13's
 * arc pair.  +8 bytes per composed arc.  Unknown flag bits: FST_E_INVALID_ARG. */
/* FST_COMPOSE_EPS_FILTER (R25): C is
 * the trim product over TRIPLES (a, b, f), f in {0 MATCH, 1 A_EPS, 2 B_EPS}, with the moves
 *     MATCH     e_a x e_b, olabel(e_a) == ilabel(e_b) != eps, from any f -> (dst e_a, dst e_b, 0)
 *     EPS-BOTH  e_a x e_b, olabel(e_a) == ilabel(e_b) == eps, only from f = 0 -> (dst, dst, 0)
 *     EPS-A     e_a with olabel eps, B stays, from f in {0, 1} -> (dst e_a, u_b, 1)
 *     EPS-B     e_b with ilabel eps, A stays, from f in {0, 2} -> (u_a, dst e_b, 2)
 * (labels and weights as M1 / M2 / M3 above); start triples (s_a, s_b, 0), accept triples
 * (f_a, f_b, any f).  Every matched path pair of Eq. (1) then yields exactly ONE
 * composed path, so log-semiring scores are exact with eps on both tapes.  pair_a / pair_b / pair_f
 * (fst_info, fst_copy_pair_f_to_host) give every state's triple; state numbering is ascending
 * (a, f, b).  Costs two passes of the binary kernels (A~ o F, then o B~; filter.cu) over a pair space
 * of about 3 V_A x V_B.  Requires labels < 2^24 and E + V < 2^31 per input (FST_E_CAPACITY).
 * Combines with FST_COMPOSE_PROVENANCE (arc_a / arc_b index the original A and B arcs). */
fst_status fst_compose_ex(fst_handle a, fst_handle b, uint32_t flags, void* stream, fst_handle* c);
fst_status fst_compose_batch_ex(int32_t n, const fst_handle* a, const fst_handle* b, uint32_t flags,
                                void* stream, fst_handle* c);

/* Copies pair_f [V] of a handle composed with FST_COMPOSE_EPS_FILTER into a HOST int32 buffer.
 * FST_E_INVALID_ARG for any other handle.  Synchronous. */
fst_status fst_copy_pair_f_to_host(fst_handle c, void* stream, int32_t* pair_f);

/* N-way composition: *c = (((g[0] o g[1]) o g[2]) ... o g[n-1]),
 * a left fold of trimmed compositions (each step filtered when flags has FST_COMPOSE_EPS_FILTER;
 * FST_COMPOSE_PROVENANCE is not supported here: FST_E_INVALID_ARG).  n >= 2; intermediates are freed.
 * The result's pair_a indexes the states of the previous fold step, pair_b the states of g[n-1]. */
fst_status fst_compose_chain(int32_t n, const fst_handle* g, uint32_t flags, void* stream, fst_handle* c);

/* Copies provenance arcs [first, first+count) of a composed handle into HOST int32 buffers (either
 * may be NULL).  FST_E_INVALID_ARG if the handle has no provenance or the range is out of bounds. */
fst_status fst_copy_provenance_to_host(fst_handle c, void* stream, int64_t first, int64_t count,
                                       int32_t* arc_a, int32_t* arc_b);

/* Gradient scatter through the composition.  Every composed weight is
 * w_c = w_a + w_b (M1) or a copy of w_a (M2) / w_b (M3), so dL/dw_a[i] = sum of dL/dw_c over the
 * arcs of C whose arc_a is i, and likewise for B.  grad_c [E_C] is read, grad_a [E_A] and grad_b
 * [E_B] are ACCUMULATED into (+=; either may be NULL).  All three are DEVICE float arrays; n_a and
 * n_b are their lengths (checked against the largest index, FST_E_INVALID_ARG if too short).
 * Needs a handle composed with FST_COMPOSE_PROVENANCE.  The per-element summation order is not
 * fixed (float atomics): results agree with an exact sum to within E_C-term rounding.
 * Asynchronous on `stream`. */
fst_status fst_grad_scatter(fst_handle c, const float* grad_c, float* grad_a, int64_t n_a, float* grad_b,
                            int64_t n_b, void* stream);

/* Forward score of an ACYCLIC graph in the log semiring (PAPER.md:368-370,
 * semiring PAPER.md:89-91): alpha(v) = logsumexp([0 if v is a start state] + {alpha(u) + w(e) :
 * e = u -> v}), *total = logsumexp of alpha over the accept states (-inf if none is reachable; an
 * empty graph gives -inf).  total: HOST double (required).  alpha: optional DEVICE double array
 * [num_states] that receives alpha (NULL to skip).  Works on any handle (composed or created).
 * Float64 throughout; the fold order of a state's in-arcs is not fixed, so results agree with an
 * exact evaluation to float64 rounding.  A cyclic graph returns FST_E_INVALID_GRAPH (the sum over
 * paths is an infinite series).  Synchronises `stream`. */
fst_status fst_forward_score(fst_handle h, void* stream, double* total, double* alpha);

/* Releases a handle and its device memory.  NULL-safe. */
void fst_free(fst_handle h);

/* Fills *v with the handle's sizes and device pointers. */
fst_status fst_info(fst_handle h, fst_view* v);

/* Copies a handle's arrays into caller-provided HOST buffers sized from fst_info (any pointer may
 * be NULL to skip that array; pair_a/pair_b only for composed handles).  Synchronous. */
fst_status fst_copy_to_host(fst_handle h, void* stream, int64_t* row_ptr, int32_t* ilabel,
                            int32_t* olabel, int32_t* dst, float* weight, uint8_t* is_start,
                            uint8_t* is_accept, int32_t* pair_a, int32_t* pair_b);

/* Copies arcs [first, first+count) of a handle into HOST buffers (any may be NULL).  Synchronous. */
fst_status fst_copy_arcs_to_host(fst_handle h, void* stream, int64_t first, int64_t count, int32_t* ilabel,
                                 int32_t* olabel, int32_t* dst, float* weight);

/* Statistics of the composition that produced handle c (composed handles only). */
fst_status fst_get_stats(fst_handle c, fst_compose_stats* s);

/* Debug accessor for the §3.2 adjacency arrays (Fig. 1 golden test): role 0 = in-arcs grouped by
 * destination (inArcOffset / inArcs), role 1 = out-arcs grouped by source.
 * Within a node, arcs are sorted by the label the view matches on (olabel for in-view... see
 * DESIGN.md) and then by arc index.  offsets [V+1], arc_ids [E], HOST buffers. */
fst_status fst_adjacency(fst_handle h, int32_t role, int32_t match_on_olabel, int64_t* offsets,
                         int64_t* arc_ids);

/* Frontier size of every BFS level of the call that produced composed handle c (stage 1 = backward
 * co-accessibility BFS, stage 2 = forward BFS; the Fig. 2 round profile).  Writes
 * min(cap, levels) entries to the HOST array `sizes` and returns the number of levels (or -1). */
int32_t fst_level_sizes(fst_handle c, int32_t stage, int64_t* sizes, int32_t cap);

/* ---- Sharded single composition over several GPUs ----------------------------
 * Ownership by state-pair block: the pair space is cut into 1024-pair blocks (32 columns of one A
 * state's row), block id = a * ceil(V_B/1024) + (b / 1024), and rank r owns the blocks with
 * id % world == r -- every row (every BFS level of a trellis-shaped composition) is spread over all
 * ranks.  Each BFS level every rank expands its own frontier pairs; pairs found in other ranks'
 * blocks are delivered to their owners (the OUT bitmap words of each peer's blocks packed into one
 * slice per peer, exchanged with grouped NCCL send/recv = all-to-all) and claimed there; R and V are
 * replicated after each stage (NCCL all-reduce, sum of disjoint bits).  States are numbered
 * OWNER-MAJOR (rank 0's states by ascending key, then rank 1's, ...): rank r's result handle holds
 * one contiguous id range (shard_info.state_offset) with GLOBAL state ids in dst; row_ptr is local
 * to the shard.  Concatenating the shards in rank order gives a valid CSR of the whole composition,
 * equal to fst_compose's after canonicalisation (identical arrays for world = 1). */
typedef struct fst_comm* fst_comm_handle;

/* 128-byte NCCL unique id, generated on one rank and broadcast by the caller (e.g. with
 * torch.distributed) before fst_comm_init.  FST_E_NCCL if NCCL cannot be loaded. */
fst_status fst_comm_unique_id(void* id128);
/* NCCL communicator over `world` ranks (one per GPU, current CUDA device). */
fst_status fst_comm_init(int32_t world, int32_t rank, const void* id128, fst_comm_handle* comm);
void fst_comm_destroy(fst_comm_handle comm); /* NULL-safe */
/* Collective: every rank calls it with the same inputs; *c_shard receives this rank's shard. */
fst_status fst_compose_sharded(fst_handle a, fst_handle b, fst_comm_handle comm, void* stream,
                               fst_handle* c_shard);
/* The same algorithm with all `world` (<= 16) shards hosted by this process on the current device
 * (the packed per-peer slices are handed over in device memory instead of NCCL): c_shards[world].
 * Used to verify the sharding on one GPU. */
fst_status fst_compose_sharded_local(fst_handle a, fst_handle b, int32_t world, void* stream,
                                     fst_handle* c_shards);

typedef struct {
  int32_t rank, world;      /* -1, 0 for unsharded handles */
  int64_t state_offset;     /* global id of this shard's first state */
  int64_t arc_offset;       /* global slot of this shard's first arc */
  int64_t total_states;     /* states / arcs of the whole composition */
  int64_t total_arcs;
} fst_shard_desc;
fst_status fst_shard_info(fst_handle c, fst_shard_desc* out);

/* Profiling: when on, fst_compose* records CUDA events per phase (fst_compose_stats) and
 * computes |R|.  Off by default. */
void fst_set_profiling(int32_t on);

/* Tile path selection for single compositions: 0 = never, 1 = automatic (pair space
 * >= 2^23 pairs and the inputs fit: degrees <= 31, labels <= 252, V_B small enough for the staged
 * tables), 2 = whenever the inputs fit, 3 = as 2 with every BFS level bottom-up, 4 = as 2 with the
 * push levels on the tile-form push kernel (tests / A-B; FSTC_TILE_PUSH=1 does the same).  The
 * environment variable FSTC_TILE sets the initial mode.  Both paths return the same graph (state
 * numbering by ascending key; arc order within a state may differ). */
void fst_set_tile_mode(int32_t mode);

/* Wave path selection: compositions whose A is topologically numbered (every arc
 * src < dst: lexicon o emissions trellises, DAGs) computed row by row (stage 1 rows descending, stage 2
 * ascending, one thread-block cluster per composition) instead of by BFS levels.  0 = never,
 * 1 = automatic (every A qualifies, rows <= 4096 per composition, A rows <= 64 arcs, B ilabels <= 252,
 * V_B < 2^24), 2 = whenever the inputs qualify, whatever their row count.  A forced tile mode (>= 2)
 * keeps single compositions on the tile path.  The environment variable FSTC_WAVE sets the initial
 * mode.  Same graph as the level path; fst_compose_stats.tile_path = 2 and levels_stage1/2 = the row
 * steps of the longest composition; no per-level sizes (fst_level_sizes returns 0 levels). */
void fst_set_wave_mode(int32_t mode);

/* Total kernels launched by this process through the library (monotone counter). */
int64_t fst_launch_count(void);

/* Thread-local message for the last non-OK status of this thread ("" if none). */
const char* fst_last_error(void);

/* Library version string. */
const char* fst_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FSTC_H_ */
