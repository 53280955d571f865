// api.cu -- the extern "C" boundary of libfstc (include/fstc.h): argument checks, error plumbing,
// handle lifetime, host copies, statistics.  All compute is in create.cu / compose.cu kernels.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <vector>

#include "fstc_handle.h"
#include "fstc_internal.cuh"
#include "nccl_dl.h"

namespace fstc {

static thread_local char g_err[512] = "";
static std::atomic<int64_t> g_launches{0};
static std::atomic<int> g_profiling{0};

void set_error(fst_status st, const char* fmt, ...) {
  (void)st;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

void count_launch(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

bool profiling_enabled() { return g_profiling.load(std::memory_order_relaxed) != 0; }

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

std::vector<int64_t>& level_sizes_slot(fst* h, int stage) { return h->level_sizes[stage == 1 ? 0 : 1]; }

fst_status compose_impl(int32_t n, const fst_handle* a, const fst_handle* b, cudaStream_t s, fst_handle* c,
                        uint32_t flags);
fst_status grad_scatter_impl(fst* c, const float* grad_c, float* grad_a, int64_t n_a, float* grad_b, int64_t n_b,
                             cudaStream_t s);
fst_status compose_sharded_impl(fst* A, fst* B, int world, fst_comm* comm, cudaStream_t s, fst_handle* c);
fst_status forward_score_impl(fst* h, cudaStream_t s, double* total, double* alpha_out);
fst_status compose_filtered_impl(int32_t n, const fst_handle* a, const fst_handle* b, cudaStream_t s, fst_handle* c,
                                 uint32_t flags);
fst_status compose_chain_impl(int32_t n, const fst_handle* g, uint32_t flags, cudaStream_t s, fst_handle* out);
void tile_mode_set(int mode);
void wave_mode_set(int mode);

fst_status device_ready() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    set_error(FST_E_CUDA, "no usable CUDA device (%s); libfstc has no CPU fallback", cudaGetErrorString(e));
    return FST_E_CUDA;
  }
  // One device per process (the multi-GPU design is one process per GPU): the library's buffer
  // cache, level scratch, capture stream, grid sizes and kernel attributes are per-process state set
  // up on the first device used, so calls made while another device is current are rejected.
  {
    static int first_dev = -1;
    int cur = 0;
    cudaGetDevice(&cur);
    if (first_dev < 0) first_dev = cur;
    if (cur != first_dev) {  // NOLINT
      set_error(FST_E_INVALID_ARG, "libfstc is bound to CUDA device %d (first use); device %d is current -- "
                "use one process per GPU", first_dev, cur);
      return FST_E_INVALID_ARG;
    }
  }
  static bool pool_done = false;
  if (!pool_done) {  // keep freed stream-ordered memory in the pool (repeat compositions reuse it)
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    pool_done = true;
  }
  return FST_OK;
}

}  // namespace fstc

using namespace fstc;

extern "C" {

fst_status fst_compose_ex(fst_handle a, fst_handle b, uint32_t flags, void* stream, fst_handle* c) {
  if (!a || !b || !c) {
    set_error(FST_E_INVALID_ARG, "fst_compose: NULL argument");
    return FST_E_INVALID_ARG;
  }
  if (flags & ~(FST_COMPOSE_PROVENANCE | FST_COMPOSE_EPS_FILTER)) {
    set_error(FST_E_INVALID_ARG, "fst_compose_ex: unknown flag bits 0x%x", flags);
    return FST_E_INVALID_ARG;
  }
  fst_status st = device_ready();
  if (st) return st;
  if (flags & FST_COMPOSE_EPS_FILTER) return compose_filtered_impl(1, &a, &b, (cudaStream_t)stream, c, flags);
  return compose_impl(1, &a, &b, (cudaStream_t)stream, c, flags);
}

fst_status fst_compose(fst_handle a, fst_handle b, void* stream, fst_handle* c) {
  return fst_compose_ex(a, b, 0u, stream, c);
}

fst_status fst_compose_batch_ex(int32_t n, const fst_handle* a, const fst_handle* b, uint32_t flags, void* stream,
                                fst_handle* c) {
  if (n < 0 || (n > 0 && (!a || !b || !c))) {
    set_error(FST_E_INVALID_ARG, "fst_compose_batch: bad arguments (n=%d)", n);
    return FST_E_INVALID_ARG;
  }
  if (flags & ~(FST_COMPOSE_PROVENANCE | FST_COMPOSE_EPS_FILTER)) {
    set_error(FST_E_INVALID_ARG, "fst_compose_batch_ex: unknown flag bits 0x%x", flags);
    return FST_E_INVALID_ARG;
  }
  if (n == 0) return FST_OK;
  fst_status st = device_ready();
  if (st) return st;
  for (int i = 0; i < n; ++i)
    if (!a[i] || !b[i]) {
      set_error(FST_E_INVALID_ARG, "fst_compose_batch: NULL handle at %d", i);
      return FST_E_INVALID_ARG;
    }
  if (flags & FST_COMPOSE_EPS_FILTER) return compose_filtered_impl(n, a, b, (cudaStream_t)stream, c, flags);
  return compose_impl(n, a, b, (cudaStream_t)stream, c, flags);
}

fst_status fst_compose_batch(int32_t n, const fst_handle* a, const fst_handle* b, void* stream, fst_handle* c) {
  return fst_compose_batch_ex(n, a, b, 0u, stream, c);
}

fst_status fst_copy_provenance_to_host(fst_handle c, void* stream, int64_t first, int64_t count, int32_t* arc_a,
                                       int32_t* arc_b) {
  if (!c || !c->arc_a || first < 0 || count < 0 || first + count > c->E) {
    set_error(FST_E_INVALID_ARG, "fst_copy_provenance_to_host: no provenance or bad range");
    return FST_E_INVALID_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (count > 0) {
    if (arc_a) FSTC_CUDA_TRY(cudaMemcpyAsync(arc_a, c->arc_a + first, 4 * count, cudaMemcpyDeviceToHost, s));
    if (arc_b) FSTC_CUDA_TRY(cudaMemcpyAsync(arc_b, c->arc_b + first, 4 * count, cudaMemcpyDeviceToHost, s));
  }
  FSTC_CUDA_TRY(cudaStreamSynchronize(s));
  return FST_OK;
}

fst_status fst_copy_pair_f_to_host(fst_handle c, void* stream, int32_t* pair_f) {
  if (!c || !c->pair_f || (c->V > 0 && !pair_f)) {
    set_error(FST_E_INVALID_ARG, "fst_copy_pair_f_to_host: not an eps-filtered composition or NULL buffer");
    return FST_E_INVALID_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (c->V > 0) FSTC_CUDA_TRY(cudaMemcpyAsync(pair_f, c->pair_f, 4 * (size_t)c->V, cudaMemcpyDeviceToHost, s));
  FSTC_CUDA_TRY(cudaStreamSynchronize(s));
  return FST_OK;
}

fst_status fst_compose_chain(int32_t n, const fst_handle* g, uint32_t flags, void* stream, fst_handle* c) {
  if (!c || n < 2 || !g) {
    set_error(FST_E_INVALID_ARG, "fst_compose_chain: need n >= 2 handles and an output");
    return FST_E_INVALID_ARG;
  }
  *c = nullptr;
  for (int i = 0; i < n; ++i)
    if (!g[i]) {
      set_error(FST_E_INVALID_ARG, "fst_compose_chain: NULL handle at %d", i);
      return FST_E_INVALID_ARG;
    }
  if (flags & ~FST_COMPOSE_EPS_FILTER) {
    set_error(FST_E_INVALID_ARG, "fst_compose_chain: unsupported flag bits 0x%x", flags);
    return FST_E_INVALID_ARG;
  }
  fst_status st = device_ready();
  if (st) return st;
  return compose_chain_impl(n, g, flags, (cudaStream_t)stream, c);
}

fst_status fst_grad_scatter(fst_handle c, const float* grad_c, float* grad_a, int64_t n_a, float* grad_b,
                            int64_t n_b, void* stream) {
  fst_status st = device_ready();
  if (st) return st;
  return grad_scatter_impl(c, grad_c, grad_a, n_a, grad_b, n_b, (cudaStream_t)stream);
}

fst_status fst_forward_score(fst_handle h, void* stream, double* total, double* alpha) {
  if (!h || !total) {
    set_error(FST_E_INVALID_ARG, "fst_forward_score: NULL argument");
    return FST_E_INVALID_ARG;
  }
  fst_status st = device_ready();
  if (st) return st;
  return forward_score_impl(h, (cudaStream_t)stream, total, alpha);
}

void fst_free(fst_handle h) {
  if (!h) return;
  // stream-ordered release: every buffer's stream first waits for the asynchronous work other streams
  // still run on this handle (fst_grad_scatter on a caller stream)
  for (cudaEvent_t ev : h->use_events) {
    for (auto& b : h->buffers)
      if (b) cudaStreamWaitEvent(b->stream, ev, 0);
    cudaEventDestroy(ev);
  }
  delete h;
}

fst_status fst_info(fst_handle h, fst_view* v) {
  if (!h || !v) {
    set_error(FST_E_INVALID_ARG, "fst_info: NULL argument");
    return FST_E_INVALID_ARG;
  }
  v->num_states = h->V;
  v->num_arcs = h->E;
  v->row_ptr = h->row_ptr;
  v->ilabel = h->ilabel;
  v->olabel = h->olabel;
  v->dst = h->dst;
  v->weight = h->weight;
  v->is_start = h->is_start;
  v->is_accept = h->is_accept;
  v->pair_a = h->composed ? h->pair_a : nullptr;
  v->pair_b = h->composed ? h->pair_b : nullptr;
  v->arc_a = h->arc_a;
  v->arc_b = h->arc_b;
  v->pair_f = h->pair_f;
  return FST_OK;
}

fst_status fst_copy_to_host(fst_handle h, void* stream, int64_t* row_ptr, int32_t* ilabel, int32_t* olabel,
                            int32_t* dst, float* weight, uint8_t* is_start, uint8_t* is_accept, int32_t* pair_a,
                            int32_t* pair_b) {
  if (!h) {
    set_error(FST_E_INVALID_ARG, "fst_copy_to_host: NULL handle");
    return FST_E_INVALID_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t V = h->V, E = h->E;
#define CPY(dst_, src_, bytes_) \
  if ((dst_) && (bytes_) > 0) FSTC_CUDA_TRY(cudaMemcpyAsync(dst_, src_, bytes_, cudaMemcpyDeviceToHost, s));
  CPY(row_ptr, h->row_ptr, 8 * (V + 1));
  CPY(ilabel, h->ilabel, 4 * E);
  CPY(olabel, h->olabel, 4 * E);
  CPY(dst, h->dst, 4 * E);
  CPY(weight, h->weight, 4 * E);
  CPY(is_start, h->is_start, V);
  CPY(is_accept, h->is_accept, V);
  if (h->composed) {
    CPY(pair_a, h->pair_a, 4 * V);
    CPY(pair_b, h->pair_b, 4 * V);
  }
#undef CPY
  FSTC_CUDA_TRY(cudaStreamSynchronize(s));
  return FST_OK;
}

fst_status fst_copy_arcs_to_host(fst_handle h, void* stream, int64_t first, int64_t count, int32_t* ilabel,
                                 int32_t* olabel, int32_t* dst, float* weight) {
  if (!h || first < 0 || count < 0 || first + count > h->E) {
    set_error(FST_E_INVALID_ARG, "fst_copy_arcs_to_host: bad range");
    return FST_E_INVALID_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (count > 0) {
    if (ilabel) FSTC_CUDA_TRY(cudaMemcpyAsync(ilabel, h->ilabel + first, 4 * count, cudaMemcpyDeviceToHost, s));
    if (olabel) FSTC_CUDA_TRY(cudaMemcpyAsync(olabel, h->olabel + first, 4 * count, cudaMemcpyDeviceToHost, s));
    if (dst) FSTC_CUDA_TRY(cudaMemcpyAsync(dst, h->dst + first, 4 * count, cudaMemcpyDeviceToHost, s));
    if (weight) FSTC_CUDA_TRY(cudaMemcpyAsync(weight, h->weight + first, 4 * count, cudaMemcpyDeviceToHost, s));
  }
  FSTC_CUDA_TRY(cudaStreamSynchronize(s));
  return FST_OK;
}

fst_status fst_get_stats(fst_handle c, fst_compose_stats* s) {
  if (!c || !s || !c->composed) {
    set_error(FST_E_INVALID_ARG, "fst_get_stats: need a composed handle");
    return FST_E_INVALID_ARG;
  }
  *s = c->stats;
  return FST_OK;
}

int32_t fst_level_sizes(fst_handle c, int32_t stage, int64_t* sizes, int32_t cap) {
  if (!c || !c->composed || (stage != 1 && stage != 2)) return -1;
  const std::vector<int64_t>& v = level_sizes_slot(c, stage);
  for (int32_t i = 0; i < cap && i < (int32_t)v.size(); ++i) sizes[i] = v[i];
  return (int32_t)v.size();
}

fst_status fst_adjacency(fst_handle h, int32_t role, int32_t match_on_olabel, int64_t* offsets, int64_t* arc_ids) {
  if (!h || !offsets || (h->E > 0 && !arc_ids) || (role != 0 && role != 1)) {
    set_error(FST_E_INVALID_ARG, "fst_adjacency: bad arguments");
    return FST_E_INVALID_ARG;
  }
  if (!h->has_views) {
    set_error(FST_E_INVALID_ARG, "fst_adjacency: handle has no views (composed handles build them on use)");
    return FST_E_INVALID_ARG;
  }
  int k = role == 0 ? (match_on_olabel ? kInByOlabel : kInByIlabel) : (match_on_olabel ? kOutByOlabel : kOutByIlabel);
  std::vector<int32_t> off(h->V + 1), arc(h->E);
  FSTC_CUDA_TRY(cudaMemcpy(off.data(), h->views[k].off, 4 * (h->V + 1), cudaMemcpyDeviceToHost));
  if (h->E) FSTC_CUDA_TRY(cudaMemcpy(arc.data(), h->views[k].arc, 4 * h->E, cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i <= h->V; ++i) offsets[i] = off[i];
  for (int64_t i = 0; i < h->E; ++i) arc_ids[i] = arc[i];
  return FST_OK;
}

fst_status fst_comm_unique_id(void* id128) {
  if (!id128) {
    set_error(FST_E_INVALID_ARG, "fst_comm_unique_id: NULL");
    return FST_E_INVALID_ARG;
  }
  const NcclApi* nc = nccl_api();
  if (!nc) return FST_E_NCCL;
  ncclUniqueId id;
  int r = nc->GetUniqueId(&id);
  if (r) {
    set_error(FST_E_NCCL, "ncclGetUniqueId failed: %s", nc->GetErrorString ? nc->GetErrorString(r) : "?");
    return FST_E_NCCL;
  }
  memcpy(id128, &id, sizeof(id));
  return FST_OK;
}

fst_status fst_comm_init(int32_t world, int32_t rank, const void* id128, fst_comm_handle* comm) {
  if (!id128 || !comm || world < 1 || rank < 0 || rank >= world) {
    set_error(FST_E_INVALID_ARG, "fst_comm_init: bad arguments");
    return FST_E_INVALID_ARG;
  }
  *comm = nullptr;
  fst_status st = device_ready();
  if (st) return st;
  const NcclApi* nc = nccl_api();
  if (!nc) return FST_E_NCCL;
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  fst_comm* c = new fst_comm();
  int r = nc->CommInitRank(&c->comm, world, id, rank);
  if (r) {
    delete c;
    set_error(FST_E_NCCL, "ncclCommInitRank failed: %s", nc->GetErrorString ? nc->GetErrorString(r) : "?");
    return FST_E_NCCL;
  }
  c->world = world;
  c->rank = rank;
  *comm = c;
  return FST_OK;
}

void fst_comm_destroy(fst_comm_handle comm) {
  if (!comm) return;
  const NcclApi* nc = nccl_api();
  if (nc && comm->comm) nc->CommDestroy(comm->comm);
  delete comm;
}

fst_status fst_compose_sharded(fst_handle a, fst_handle b, fst_comm_handle comm, void* stream, fst_handle* c) {
  if (!a || !b || !comm || !c) {
    set_error(FST_E_INVALID_ARG, "fst_compose_sharded: NULL argument");
    return FST_E_INVALID_ARG;
  }
  *c = nullptr;
  fst_status st = device_ready();
  if (st) return st;
  return compose_sharded_impl(a, b, comm->world, comm, (cudaStream_t)stream, c);
}

fst_status fst_compose_sharded_local(fst_handle a, fst_handle b, int32_t world, void* stream, fst_handle* c) {
  if (!a || !b || !c || world < 1) {
    set_error(FST_E_INVALID_ARG, "fst_compose_sharded_local: bad arguments");
    return FST_E_INVALID_ARG;
  }
  for (int i = 0; i < world; ++i) c[i] = nullptr;
  fst_status st = device_ready();
  if (st) return st;
  return compose_sharded_impl(a, b, world, nullptr, (cudaStream_t)stream, c);
}

fst_status fst_shard_info(fst_handle c, fst_shard_desc* out) {
  if (!c || !out) {
    set_error(FST_E_INVALID_ARG, "fst_shard_info: NULL argument");
    return FST_E_INVALID_ARG;
  }
  out->rank = c->shard_rank;
  out->world = c->shard_world;
  out->state_offset = c->shard_state_offset;
  out->arc_offset = c->shard_arc_offset;
  out->total_states = c->shard_rank >= 0 ? c->shard_total_states : c->V;
  out->total_arcs = c->shard_rank >= 0 ? c->shard_total_arcs : c->E;
  return FST_OK;
}

void fst_set_profiling(int32_t on) { g_profiling.store(on ? 1 : 0); }

void fst_set_tile_mode(int32_t mode) { fstc::tile_mode_set(mode); }

void fst_set_wave_mode(int32_t mode) { fstc::wave_mode_set(mode); }

int64_t fst_launch_count(void) { return g_launches.load(); }

const char* fst_last_error(void) { return g_err; }

const char* fst_version(void) { return "fstc 0.1 (sm_100a)"; }

}  // extern "C"
