// filter.cu -- the eps-filtered composition and N-way chains (rank 4), built
// on the binary composition kernels of compose.cu.
//
// eps filter.  The paper claims eps support but its Algorithm 1 has no
// redundancy filter: under reading N1 a matched path pair with eps runs on both tapes yields
// Delannoy-many composed paths.  The three-state filter (DESIGN.md
// §2 R25) removes the duplicates: states are triples (a, b, f), f in {0 MATCH, 1 A_EPS, 2 B_EPS};
// MATCH moves (o_a == i_b != eps) from any f -> 0, EPS-BOTH (o_a == i_b == eps) only from 0 -> 0,
// EPS-A (o_a = eps, B stays) from {0,1} -> 1, EPS-B (i_b = eps, A stays) from {0,2} -> 2.
//
// B200 design: no new BFS kernels.  The filtered product is the eps-FREE three-way product
// A~ o F o B~, composed as two passes of the existing level-synchronous kernels:
//   A~ = A with every output eps relabelled E2 and a self-loop  eps:E1  (weight -0.0) on every state
//   B~ = B with every input  eps relabelled E1 and a self-loop  E2:eps  (weight -0.0) on every state
//   F  = 3 states, all final, start 0:   x:x (every real label x) from 0, 1, 2 -> 0 (MATCH);
//        E2:E1 from 0 -> 0 (EPS-BOTH);  E2:E2 from 0, 1 -> 1 (EPS-A);  E1:E1 from 0, 2 -> 2 (EPS-B)
// (E1 = L, E2 = L + 1, L = 1 + the largest real label on A's output / B's input tape.)  A path of
// A~ o F o B~ spells exactly one filtered move per step: A~'s self-loop (A stays) can only meet F's
// E1:E1 arcs and B's relabelled eps-input arcs (EPS-B), B~'s self-loop only F's E2:E2 arcs and A's
// eps-output arcs (EPS-A); E2:E1 pairs A's and B's eps arcs (EPS-BOTH).  Nothing on A~'s output or
// B~'s input tape is eps any more, so both passes use only M1 moves.  -0.0 is the exact additive
// identity of IEEE binary32 RN-even (x + -0.0 == x bitwise, including x = -0.0), so every composed
// weight is the same single add (or bit copy) as the direct definition.  C1 = trim(A~ o F) keeps
// every (a, f) on an accepted triple path (F is all-final), so trim(C1 o B~) = the trim filtered
// product; state (c1, b) maps to the triple (C1.pair_a[c1], b, C1.pair_b[c1]).
//
// Shortcut: when no A arc has an eps output and no B arc an eps input, every move is MATCH and the
// filtered graph is the plain composition with f = 0 (one pass, no marked copies).
//
// N-way ("N-way composition instead of just two inputs"): a left fold
// ((G0 o G1) o G2) o ... of full trimmed compositions; intermediates are freed as the fold goes.
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <vector>

#include "fstc_handle.h"
#include "fstc_internal.cuh"

namespace fstc {

fst_status compose_impl(int32_t n, const fst_handle* a, const fst_handle* b, cudaStream_t s, fst_handle* c,
                        uint32_t flags);
fst_status ensure_views(fst* h, cudaStream_t s);

namespace {

inline unsigned nblk(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

// Marked copy of one side.  Row v of the output holds v's arcs (relabelled) then one self-loop, so
// output arc j of input arc e (source v) is j = e + v; map[j] = e, or -1 for the self-loop.
//   side 0 (A~): olabel eps -> relabel; loop  eps : loop_lab
//   side 1 (B~): ilabel eps -> relabel; loop  loop_lab : eps
__global__ void k_mark_arcs(int32_t V, int64_t E, const int64_t* __restrict__ rp, const int32_t* __restrict__ il,
                            const int32_t* __restrict__ ol, const int32_t* __restrict__ dst,
                            const float* __restrict__ w, int side, int32_t relabel, int32_t* __restrict__ il2,
                            int32_t* __restrict__ ol2, int32_t* __restrict__ dst2, float* __restrict__ w2,
                            int32_t* __restrict__ map) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    int32_t lo = 0, hi = V - 1;  // source state: largest v with rp[v] <= e
    while (lo < hi) {
      const int32_t mid = (lo + hi + 1) >> 1;
      if (rp[mid] <= e) lo = mid; else hi = mid - 1;
    }
    const int64_t j = e + lo;
    int32_t a = il[e], b = ol[e];
    if (side == 0 && b == FST_EPS) b = relabel;
    if (side == 1 && a == FST_EPS) a = relabel;
    il2[j] = a;
    ol2[j] = b;
    dst2[j] = dst[e];
    w2[j] = w[e];
    map[j] = (int32_t)e;
  }
}

__global__ void k_mark_loops(int32_t V, int64_t E, const int64_t* __restrict__ rp, int side, int32_t loop_lab,
                             int64_t* __restrict__ rp2, int32_t* __restrict__ il2, int32_t* __restrict__ ol2,
                             int32_t* __restrict__ dst2, float* __restrict__ w2, int32_t* __restrict__ map) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v <= V; v += (int64_t)gridDim.x * blockDim.x) {
    rp2[v] = rp[v] + v;
    if (v == V) continue;
    const int64_t j = rp[v + 1] + v;  // after the row's arcs
    il2[j] = side == 0 ? FST_EPS : loop_lab;
    ol2[j] = side == 0 ? loop_lab : FST_EPS;
    dst2[j] = (int32_t)v;
    w2[j] = -0.0f;  // exact additive identity: x + (-0.0) == x bitwise
    map[j] = -1;
  }
}

// Triple of every state of C = C1 o B~: (a, f) = (C1.pair_a, C1.pair_b) of its C1 state.
__global__ void k_filter_triples(int32_t V, const int32_t* __restrict__ c1_pa, const int32_t* __restrict__ c1_pb,
                                 int32_t* __restrict__ pair_a, int32_t* __restrict__ pair_f) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < V; s += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c1 = pair_a[s];
    pair_a[s] = c1_pa[c1];
    pair_f[s] = c1_pb[c1];
  }
}

// Provenance through the chain: C arc -> (C1 arc, B~ arc); C1 arc -> A~ arc; marked arcs -> input
// arcs (-1 for the self-loops, i.e. the side that stays).
__global__ void k_filter_prov(int64_t E, int32_t* __restrict__ arc_a, int32_t* __restrict__ arc_b,
                              const int32_t* __restrict__ c1_arc_a, const int32_t* __restrict__ amap,
                              const int32_t* __restrict__ bmap) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < E; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t x = arc_a[k], y = arc_b[k];  // both >= 0: every move of both passes is M1
    arc_a[k] = amap[c1_arc_a[x]];
    arc_b[k] = bmap[y];
  }
}

__global__ void k_any_eps(const int32_t* __restrict__ lab, int64_t E, int32_t* __restrict__ flag) {
  bool hit = false;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
    hit |= lab[e] == FST_EPS;
  if (__any_sync(0xffffffffu, hit) && (threadIdx.x & 31) == 0) *flag = 1;
}

struct Marked {
  fst_handle h = nullptr;
  BufferPtr map;  // [E+V] marked arc -> input arc (-1 = self-loop)
};

fst_status make_marked(fst* g, int side, int32_t relabel, int32_t loop_lab, cudaStream_t s, Marked* out) {
  const int32_t V = g->V;
  const int64_t E2 = g->E + V;
  if (E2 >= INT32_MAX) {
    set_error(FST_E_CAPACITY, "eps filter: E + V of an input must be < 2^31");
    return FST_E_CAPACITY;
  }
  BufferPtr tmp;
  const size_t n8 = ((size_t)(V + 1) * 8 + 255) & ~size_t(255), n4 = ((size_t)E2 * 4 + 255) & ~size_t(255);
  fst_status st = alloc_buffer(n8 + 4 * n4 + 512, s, &tmp);
  if (st) return st;
  st = alloc_buffer(n4 + 256, s, &out->map);
  if (st) return st;
  char* p = (char*)tmp->ptr;
  int64_t* rp2 = (int64_t*)p;
  int32_t* il2 = (int32_t*)(p + n8);
  int32_t* ol2 = (int32_t*)(p + n8 + n4);
  int32_t* dst2 = (int32_t*)(p + n8 + 2 * n4);
  float* w2 = (float*)(p + n8 + 3 * n4);
  uint8_t* flags = (uint8_t*)(p + n8 + 4 * n4);  // unused placeholder when V == 0
  int32_t* map = (int32_t*)out->map->ptr;
  if (g->E > 0) {
    k_mark_arcs<<<nblk(g->E, 256), 256, 0, s>>>(V, g->E, g->row_ptr, g->ilabel, g->olabel, g->dst, g->weight, side,
                                                relabel, il2, ol2, dst2, w2, map);
    FSTC_LAUNCH_CHECK();
  }
  k_mark_loops<<<nblk((int64_t)V + 1, 256), 256, 0, s>>>(V, g->E, g->row_ptr, side, loop_lab, rp2, il2, ol2, dst2, w2,
                                                         map);
  FSTC_LAUNCH_CHECK();
  fst_desc d;
  d.num_states = V;
  d.num_arcs = E2;
  d.row_ptr = rp2;
  d.ilabel = il2;
  d.olabel = ol2;
  d.dst = dst2;
  d.weight = w2;
  d.is_start = V ? g->is_start : flags;
  d.is_accept = V ? g->is_accept : flags;
  d.memory = FST_MEM_DEVICE;
  return fst_create(&d, s, &out->h);  // copies + validates + builds the label-sorted views
}

// The filter transducer F for real labels 0..L-1 (E1 = L, E2 = L + 1), weights -0.0.
fst_status make_filter(int32_t L, cudaStream_t s, fst_handle* out) {
  const int32_t E1 = L, E2 = L + 1;
  std::vector<int64_t> rp(4, 0);
  std::vector<int32_t> il, ol, dst;
  auto arc = [&](int32_t i, int32_t o, int32_t d) { il.push_back(i); ol.push_back(o); dst.push_back(d); };
  for (int f = 0; f < 3; ++f) {
    for (int32_t x = 0; x < L; ++x) arc(x, x, 0);  // MATCH from any f -> 0
    if (f == 0) arc(E2, E1, 0);                      // EPS-BOTH: A's eps output meets B's eps input
    if (f != 2) arc(E2, E2, 1);                      // EPS-A (A moves, B~ self-loop) from {0, 1} -> 1
    if (f != 1) arc(E1, E1, 2);                      // EPS-B (A~ self-loop, B moves) from {0, 2} -> 2
    rp[f + 1] = (int64_t)il.size();
  }
  std::vector<float> w(il.size(), -0.0f);
  const uint8_t st[3] = {1, 0, 0}, ac[3] = {1, 1, 1};
  fst_desc d;
  d.num_states = 3;
  d.num_arcs = (int64_t)il.size();
  d.row_ptr = rp.data();
  d.ilabel = il.data();
  d.olabel = ol.data();
  d.dst = dst.data();
  d.weight = w.data();
  d.is_start = st;
  d.is_accept = ac;
  d.memory = FST_MEM_HOST;
  return fst_create(&d, s, out);
}

}  // namespace

// Does any arc of a side carry eps on the matched tape (A: olabel, B: ilabel)?  Without eps there
// the filter never leaves MATCH and the filtered graph is the plain one with f = 0.
fst_status matched_tape_has_eps(const fst* g, bool a_side, cudaStream_t s, bool* out) {
  *out = false;
  if (g->E == 0) return FST_OK;
  BufferPtr fb;
  fst_status st = alloc_buffer(256, s, &fb);
  if (st) return st;
  int32_t* flag = (int32_t*)fb->ptr;
  FSTC_CUDA_TRY(cudaMemsetAsync(flag, 0, 4, s));
  k_any_eps<<<std::min(nblk(g->E, 256), 1184u), 256, 0, s>>>(a_side ? g->olabel : g->ilabel, g->E, flag);
  FSTC_LAUNCH_CHECK();
  int32_t h = 0;
  FSTC_CUDA_TRY(cudaMemcpyAsync(&h, flag, 4, cudaMemcpyDeviceToHost, s));
  FSTC_CUDA_TRY(cudaStreamSynchronize(s));
  *out = h != 0;
  return FST_OK;
}

fst_status compose_filtered_impl(int32_t n, const fst_handle* a, const fst_handle* b, cudaStream_t s, fst_handle* c,
                                 uint32_t flags) {
  const bool want_prov = flags & FST_COMPOSE_PROVENANCE;
  for (int i = 0; i < n; ++i) c[i] = nullptr;
  {  // eps-free matched tapes everywhere: one plain pass, f = 0 for every state
    std::map<std::pair<const fst*, bool>, bool> seen;
    bool any = false;
    for (int i = 0; i < n && !any; ++i) {
      for (int side = 0; side < 2 && !any; ++side) {
        const fst* g = side == 0 ? a[i] : b[i];
        auto key = std::make_pair(g, side == 0);
        auto it = seen.find(key);
        bool has;
        if (it != seen.end()) {
          has = it->second;
        } else {
          fst_status st = matched_tape_has_eps(g, side == 0, s, &has);
          if (st) return st;
          seen[key] = has;
        }
        any |= has;
      }
    }
    if (!any) {
      fst_status st = compose_impl(n, a, b, s, c, flags & FST_COMPOSE_PROVENANCE);
      if (st) return st;
      for (int i = 0; i < n && !st; ++i) {
        fst* h = c[i];
        BufferPtr pf;
        st = alloc_buffer((size_t)std::max<int32_t>(h->V, 1) * 4, s, &pf);
        if (st) break;
        h->pair_f = (int32_t*)pf->ptr;
        h->buffers.push_back(pf);
        h->filtered = true;
        if (h->V > 0 && cudaMemsetAsync(h->pair_f, 0, 4 * (size_t)h->V, s) != cudaSuccess) {
          set_error(FST_E_CUDA, "eps filter: memset failed");
          st = FST_E_CUDA;
        }
      }
      if (!st && cudaStreamSynchronize(s) != cudaSuccess) {
        set_error(FST_E_CUDA, "eps filter: synchronize failed");
        st = FST_E_CUDA;
      }
      if (st)
        for (int i = 0; i < n; ++i) {
          fst_free(c[i]);
          c[i] = nullptr;
        }
      return st;
    }
  }
  // marked copies are built once per distinct input handle (a batch usually repeats its B)
  std::map<std::pair<const fst*, int32_t>, Marked> amk, bmk;
  std::vector<Marked*> am(n), bm(n);
  std::map<int32_t, fst_handle> filters;
  std::vector<fst_handle> fa(n), c1(n, nullptr), am_h(n), bm_h(n);
  fst_status st = FST_OK;
  auto cleanup = [&]() {
    for (auto& kv : amk) fst_free(kv.second.h);
    for (auto& kv : bmk) fst_free(kv.second.h);
    for (auto& kv : filters) fst_free(kv.second);
    for (auto h : c1) fst_free(h);
  };
  for (int i = 0; i < n && !st; ++i) {
    st = ensure_views(a[i], s);
    if (!st) st = ensure_views(b[i], s);
    if (st) break;
    const int64_t L = (int64_t)std::max(std::max(a[i]->max_olabel, b[i]->max_ilabel), -1) + 1;
    if (L > (1 << 24)) {
      set_error(FST_E_CAPACITY, "eps filter: labels must be < 2^24 (the filter has 3 arcs per label)");
      st = FST_E_CAPACITY;
      break;
    }
    const int32_t E1 = (int32_t)L, E2 = (int32_t)L + 1;
    const auto ka = std::make_pair((const fst*)a[i], E1), kb = std::make_pair((const fst*)b[i], E1);
    if (!amk.count(ka)) st = make_marked(a[i], 0, E2, E1, s, &amk[ka]);
    if (!st && !bmk.count(kb)) st = make_marked(b[i], 1, E1, E2, s, &bmk[kb]);
    if (!st && !filters.count(E1)) {
      fst_handle f = nullptr;
      st = make_filter(E1, s, &f);
      if (!st) filters[E1] = f;
    }
    if (!st) {
      am[i] = &amk[ka];
      bm[i] = &bmk[kb];
      fa[i] = filters[E1];
      am_h[i] = am[i]->h;
      bm_h[i] = bm[i]->h;
    }
  }
  if (!st) st = compose_impl(n, am_h.data(), fa.data(), s, c1.data(), flags);
  if (!st) st = compose_impl(n, c1.data(), bm_h.data(), s, c, flags);
  for (int i = 0; i < n && !st; ++i) {
    fst* h = c[i];
    BufferPtr pf;
    st = alloc_buffer((size_t)std::max<int32_t>(h->V, 1) * 4, s, &pf);
    if (st) break;
    h->pair_f = (int32_t*)pf->ptr;
    h->buffers.push_back(pf);
    if (h->V > 0) {
      k_filter_triples<<<nblk(h->V, 256), 256, 0, s>>>(h->V, c1[i]->pair_a, c1[i]->pair_b, h->pair_a, h->pair_f);
      count_launch();
    }
    if (want_prov && h->E > 0) {
      k_filter_prov<<<nblk(h->E, 256), 256, 0, s>>>(h->E, h->arc_a, h->arc_b, c1[i]->arc_a,
                                                    (const int32_t*)am[i]->map->ptr, (const int32_t*)bm[i]->map->ptr);
      count_launch();
    }
    h->src_arcs_a = a[i]->E;
    h->src_arcs_b = b[i]->E;
    h->filtered = true;
    if (cudaGetLastError() != cudaSuccess) {
      set_error(FST_E_CUDA, "eps filter: kernel launch failed");
      st = FST_E_CUDA;
    }
  }
  if (!st) {
    cudaError_t e = cudaStreamSynchronize(s);  // c1 / marked buffers are released below
    if (e != cudaSuccess) {
      set_error(FST_E_CUDA, "eps filter: %s", cudaGetErrorString(e));
      st = FST_E_CUDA;
    }
  }
  cleanup();
  if (st) {
    for (int i = 0; i < n; ++i) {
      fst_free(c[i]);
      c[i] = nullptr;
    }
  }
  return st;
}

// Left fold over g[0..n-1]; each step is fst_compose(_ex) (filtered when FST_COMPOSE_EPS_FILTER).
fst_status compose_chain_impl(int32_t n, const fst_handle* g, uint32_t flags, cudaStream_t s, fst_handle* out) {
  *out = nullptr;
  fst_handle cur = g[0];
  for (int i = 1; i < n; ++i) {
    fst_handle next = nullptr;
    fst_status st = (flags & FST_COMPOSE_EPS_FILTER) ? compose_filtered_impl(1, &cur, &g[i], s, &next, 0u)
                                                      : compose_impl(1, &cur, &g[i], s, &next, 0u);
    if (i > 1) {  // the previous intermediate is ours
      cudaStreamSynchronize(s);
      fst_free(cur);
    }
    if (st) return st;
    cur = next;
  }
  *out = cur;
  return FST_OK;
}

}  // namespace fstc
