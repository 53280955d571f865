// create.cu -- fst_create: upload, validation and the label-sorted adjacency views (SURVEY §8(a)
// a0; the SoA transducer with in/out arc arrays and offsets of PAPER.md:172-194).
//
// Views are built on the device with a CUB-free stable LSD radix sort (4-bit digits) of the
// composite key (node << LB) | (label + 1), payload = arc index.  eps (-1) maps to 0 and therefore
// sorts first inside a node: the eps arcs of a node are a prefix of its view.
#include <stdarg.h>
#include <stdio.h>

#include <algorithm>

#include "fstc_handle.h"
#include "fstc_internal.cuh"
#include "scan.cuh"

namespace fstc {

fst_status device_ready();

namespace {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 8;
constexpr int kSortTile = kSortThreads * kSortItems;  // 2048

// ------------------------------------------------------------------ validation
// err bits: 1 row_ptr[0]!=0, 2 row_ptr decreasing, 4 row_ptr[V]!=E, 8 dst out of range,
//           16 label < -1, 32 non-finite weight, 64 flag not in {0,1}
__global__ void k_validate_states(int32_t V, int64_t E, const int64_t* __restrict__ row_ptr,
                                  const uint8_t* __restrict__ st, const uint8_t* __restrict__ ac,
                                  int32_t* __restrict__ out) {
  int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v > V) return;
  int err = 0;
  if (v == 0 && row_ptr[0] != 0) err |= 1;
  if (v == V && row_ptr[V] != E) err |= 4;
  if (v < V) {
    if (row_ptr[v + 1] < row_ptr[v]) err |= 2;
    if (st[v] > 1 || ac[v] > 1) err |= 64;
  }
  if (err) atomicOr(&out[0], err);
}

__global__ void k_validate_arcs(int32_t V, int64_t E, const int32_t* __restrict__ il,
                                const int32_t* __restrict__ ol, const int32_t* __restrict__ dst,
                                const float* __restrict__ w, int32_t* __restrict__ out) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int err = 0, mi = -1, mo = -1;
  if (e < E) {
    int32_t a = il[e], b = ol[e], d = dst[e];
    if (d < 0 || d >= V) err |= 8;
    if (a < -1 || b < -1) err |= 16;
    if (!isfinite(w[e])) err |= 32;
    mi = a;
    mo = b;
  }
  mi = max(mi, __shfl_xor_sync(0xffffffffu, mi, 16));
  mi = max(mi, __shfl_xor_sync(0xffffffffu, mi, 8));
  mi = max(mi, __shfl_xor_sync(0xffffffffu, mi, 4));
  mi = max(mi, __shfl_xor_sync(0xffffffffu, mi, 2));
  mi = max(mi, __shfl_xor_sync(0xffffffffu, mi, 1));
  mo = max(mo, __shfl_xor_sync(0xffffffffu, mo, 16));
  mo = max(mo, __shfl_xor_sync(0xffffffffu, mo, 8));
  mo = max(mo, __shfl_xor_sync(0xffffffffu, mo, 4));
  mo = max(mo, __shfl_xor_sync(0xffffffffu, mo, 2));
  mo = max(mo, __shfl_xor_sync(0xffffffffu, mo, 1));
  err |= __reduce_or_sync(0xffffffffu, (unsigned)err);
  if ((threadIdx.x & 31) == 0) {
    if (err) atomicOr(&out[0], err);
    atomicMax(&out[1], mi);
    atomicMax(&out[2], mo);
  }
}

// ------------------------------------------------------------------ arc sources
__global__ void k_arc_src(int32_t V, int64_t E, const int64_t* __restrict__ row_ptr,
                          int32_t* __restrict__ src) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  int32_t lo = 0, hi = V - 1;  // last v with row_ptr[v] <= e
  while (lo < hi) {
    int32_t mid = (lo + hi + 1) >> 1;
    if (row_ptr[mid] <= e) lo = mid; else hi = mid - 1;
  }
  src[e] = lo;
}

// ------------------------------------------------------------------ radix sort (stable LSD)
__global__ void k_make_keys(int64_t E, const int32_t* __restrict__ node, const int32_t* __restrict__ label,
                            int LB, unsigned long long* __restrict__ keys, int32_t* __restrict__ vals) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  keys[e] = ((unsigned long long)(uint32_t)node[e] << LB) | (unsigned long long)(uint32_t)(label[e] + 1);
  vals[e] = (int32_t)e;
}

__global__ void __launch_bounds__(kSortThreads) k_radix_hist(const unsigned long long* __restrict__ keys,
                                                             int64_t n, int shift, int32_t* __restrict__ hist,
                                                             int ntiles) {
  __shared__ int32_t h[16];
  if (threadIdx.x < 16) h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
#pragma unroll
  for (int k = 0; k < kSortItems; ++k) {
    int64_t i = base + (int64_t)k * kSortThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[(keys[i] >> shift) & 15], 1);
  }
  __syncthreads();
  if (threadIdx.x < 16) hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

__device__ __forceinline__ unsigned field16(const unsigned long long (&p)[4], int d) {
  return (unsigned)((p[d >> 2] >> (16 * (d & 3))) & 0xFFFFu);
}

__global__ void __launch_bounds__(kSortThreads) k_radix_scatter(
    const unsigned long long* __restrict__ kin, const int32_t* __restrict__ vin, int64_t n, int shift,
    const int64_t* __restrict__ off /* [16*ntiles] exclusive, digit-major */, int ntiles,
    unsigned long long* __restrict__ kout, int32_t* __restrict__ vout) {
  __shared__ unsigned long long sh[kSortThreads / 32 + 1];
  const int64_t base = (int64_t)blockIdx.x * kSortTile + (int64_t)threadIdx.x * kSortItems;  // blocked
  unsigned long long k[kSortItems];
  int32_t v[kSortItems];
  int d[kSortItems];
  unsigned lr[kSortItems];
  unsigned long long cnt[4] = {0, 0, 0, 0};
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    int64_t i = base + j;
    if (i < n) {
      k[j] = kin[i];
      v[j] = vin[i];
      d[j] = (int)((k[j] >> shift) & 15);
      lr[j] = field16(cnt, d[j]);
      cnt[d[j] >> 2] += 1ull << (16 * (d[j] & 3));
    } else {
      d[j] = -1;
    }
  }
  unsigned long long ex[4], tot;
#pragma unroll
  for (int q = 0; q < 4; ++q) ex[q] = block_excl_scan(cnt[q], sh, &tot);
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    if (d[j] < 0) continue;
    int64_t pos = off[(int64_t)d[j] * ntiles + blockIdx.x] + field16(ex, d[j]) + lr[j];
    kout[pos] = k[j];
    vout[pos] = v[j];
  }
}

// ------------------------------------------------------------------ view assembly
__global__ void k_gather_view(int64_t E, const int32_t* __restrict__ perm, const int32_t* __restrict__ key_src,
                              const int32_t* __restrict__ other_src, const int32_t* __restrict__ carry_src,
                              const float* __restrict__ w_src, int32_t* __restrict__ key,
                              int32_t* __restrict__ other, int32_t* __restrict__ carry, float* __restrict__ w,
                              int32_t* __restrict__ arc, int2* __restrict__ cw) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= E) return;
  int32_t e = perm[i];
  const int32_t k = key_src[e], o = other_src[e], c = carry_src[e];
  const float x = w_src[e];
  key[i] = k;
  other[i] = o;
  carry[i] = c;
  w[i] = x;
  arc[i] = e;
  cw[i] = make_int2(c, __float_as_int(x));
}

// off[v] = first sorted position whose node >= v  (node = key >> LB)
__global__ void k_view_offsets(int32_t V, int64_t E, const unsigned long long* __restrict__ keys, int LB,
                               int32_t* __restrict__ off) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > E) return;
  int64_t prev = i > 0 ? (int64_t)(keys[i - 1] >> LB) : -1;
  int64_t cur = i < E ? (int64_t)(keys[i] >> LB) : (int64_t)V;
  for (int64_t v = prev + 1; v <= cur; ++v) off[v] = (int32_t)i;
}

// items of a view: node v owns [off[v]+v, off[v+1]+v+1): sentinel, then its arcs in view order
__global__ void k_view_items(int32_t V, int64_t E, const int32_t* __restrict__ off, const int32_t* __restrict__ key,
                             const int32_t* __restrict__ other, const unsigned long long* __restrict__ keys, int LB,
                             const int2* __restrict__ cw, int2* __restrict__ ikd, int32_t* __restrict__ isrc,
                             int4* __restrict__ ikcw) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < E) {
    const int32_t v = (int32_t)(keys[i] >> LB);
    const int2 c = cw[i];
    ikd[i + v + 1] = make_int2(key[i], other[i]);
    ikcw[i + v + 1] = make_int4(key[i], other[i], c.x, c.y);
    isrc[i + v + 1] = v;
  }
  if (i < V) {
    ikd[off[i] + i] = make_int2(kSentinel, (int32_t)i);
    ikcw[off[i] + i] = make_int4(kSentinel, (int32_t)i, 0, 0);
    isrc[off[i] + i] = (int32_t)i;
  }
}

// label-major keys: ((label+1) << NB) | node, payload = view position
__global__ void k_lm_keys(int64_t E, const unsigned long long* __restrict__ vkeys, int LB, int NB,
                          const int32_t* __restrict__ key, unsigned long long* __restrict__ out,
                          int32_t* __restrict__ vals) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= E) return;
  const unsigned long long node = vkeys[i] >> LB;
  out[i] = ((unsigned long long)(uint32_t)(key[i] + 1) << NB) | node;
  vals[i] = (int32_t)i;
}

__global__ void k_lm_flags(int64_t E, const unsigned long long* __restrict__ keys, const int32_t* __restrict__ vals,
                           int NB, const int32_t* __restrict__ other, int32_t* __restrict__ lm_other,
                           int32_t* __restrict__ lm_pos, int32_t* __restrict__ segf, int32_t* __restrict__ labf) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= E) return;
  const int32_t p = vals[i];
  lm_pos[i] = p;
  lm_other[i] = other[p];
  const unsigned long long k = keys[i];
  segf[i] = (i == 0 || k != keys[i - 1]) ? 1 : 0;
  labf[i] = (i == 0 || (k >> NB) != (keys[i - 1] >> NB)) ? 1 : 0;
}

__global__ void k_lm_scatter(int64_t E, const unsigned long long* __restrict__ keys, int NB,
                             const int32_t* __restrict__ segf, const int32_t* __restrict__ labf,
                             const int64_t* __restrict__ segi, const int64_t* __restrict__ labi,
                             int32_t* __restrict__ seg_node, int32_t* __restrict__ seg_beg,
                             int32_t* __restrict__ lab_val, int32_t* __restrict__ lab_seg) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > E) return;
  if (i == E) {
    seg_beg[segi[E]] = (int32_t)E;
    lab_seg[labi[E]] = (int32_t)segi[E];
    return;
  }
  const unsigned long long k = keys[i];
  if (segf[i]) {
    seg_node[segi[i]] = (int32_t)(k & ((1ull << NB) - 1));
    seg_beg[segi[i]] = (int32_t)i;
  }
  if (labf[i]) {
    lab_val[labi[i]] = (int32_t)(k >> NB) - 1;
    lab_seg[labi[i]] = (int32_t)segi[i];
  }
}

// start / accept lists in ascending state order (single CTA, block scan)
__global__ void __launch_bounds__(1024) k_flag_lists(int32_t V, const uint8_t* __restrict__ st,
                                                     const uint8_t* __restrict__ ac,
                                                     int32_t* __restrict__ slist, int32_t* __restrict__ alist,
                                                     int32_t* __restrict__ counts) {
  __shared__ int32_t sh[1024 / 32 + 1];
  int32_t cs = 0, ca = 0;
  for (int32_t b = 0; b < V; b += blockDim.x) {
    int32_t v = b + threadIdx.x;
    int32_t fs = v < V ? (int32_t)st[v] : 0;
    int32_t fa = v < V ? (int32_t)ac[v] : 0;
    int32_t ts, ta;
    int32_t es = block_excl_scan(fs, sh, &ts);
    int32_t ea = block_excl_scan(fa, sh, &ta);
    if (fs) slist[cs + es] = v;
    if (fa) alist[ca + ea] = v;
    cs += ts;
    ca += ta;
  }
  if (threadIdx.x == 0) {
    counts[0] = cs;
    counts[1] = ca;
  }
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

__global__ void k_view_maxdeg(int32_t V, const int32_t* __restrict__ off, int32_t* __restrict__ out) {
  int32_t m = 0;
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x)
    m = max(m, off[v + 1] - off[v]);
  m = __reduce_max_sync(0xffffffffu, (unsigned)m);
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

int bits_for(int64_t x) {  // bits to represent values in [0, x]
  int b = 0;
  while (b < 62 && (1ll << b) <= x) ++b;
  return std::max(b, 1);
}

}  // namespace

// Simple bump allocator over one buffer.
struct Carve {
  char* p;
  size_t used = 0;
  template <typename T>
  T* take(int64_t n) {
    T* r = reinterpret_cast<T*>(p + used);
    used += ((size_t)std::max<int64_t>(n, 1) * sizeof(T) + 255) & ~size_t(255);
    return r;
  }
};
template <typename T>
static size_t carve_bytes(int64_t n) {
  return ((size_t)std::max<int64_t>(n, 1) * sizeof(T) + 255) & ~size_t(255);
}

// Build the four label-sorted views of h (its CSR must be on the device).  Sync on s.
fst_status build_views(fst* h, cudaStream_t s, int32_t max_il, int32_t max_ol) {
  const int64_t E = h->E;
  const int32_t V = h->V;
  if (E > INT32_MAX - 1) {
    set_error(FST_E_CAPACITY, "views need E < 2^31 (E = %lld)", (long long)E);
    return FST_E_CAPACITY;
  }
  size_t vbytes = 0;
  for (int k = 0; k < 4; ++k)
    vbytes += carve_bytes<int32_t>(V + 1) + 4 * carve_bytes<int32_t>(E) + carve_bytes<float>(E) +
              carve_bytes<int2>(E) + carve_bytes<int2>(E + V) + carve_bytes<int32_t>(E + V) + carve_bytes<int4>(E + V) +
              4 * carve_bytes<int32_t>(E) + 2 * carve_bytes<int32_t>(E + 1);
  vbytes += 2 * carve_bytes<int32_t>(V);
  BufferPtr vb;
  fst_status st = alloc_buffer(vbytes, s, &vb);
  if (st) return st;
  h->buffers.push_back(vb);
  Carve cv{(char*)vb->ptr};
  for (int k = 0; k < 4; ++k) {
    View& w = h->views[k];
    w.off = cv.take<int32_t>(V + 1);
    w.key = cv.take<int32_t>(E);
    w.other = cv.take<int32_t>(E);
    w.carry = cv.take<int32_t>(E);
    w.arc = cv.take<int32_t>(E);
    w.w = cv.take<float>(E);
    w.cw = cv.take<int2>(E);
    w.ikd = cv.take<int2>(E + V);
    w.isrc = cv.take<int32_t>(E + V);
    w.ikcw = cv.take<int4>(E + V);
    w.lm_other = cv.take<int32_t>(E);
    w.lm_pos = cv.take<int32_t>(E);
    w.seg_node = cv.take<int32_t>(E);
    w.seg_beg = cv.take<int32_t>(E + 1);
    w.lab_val = cv.take<int32_t>(E);
    w.lab_seg = cv.take<int32_t>(E + 1);
  }
  h->start_list = cv.take<int32_t>(V);
  h->accept_list = cv.take<int32_t>(V);

  // temporaries
  const int64_t ntiles = std::max<int64_t>(1, (E + kSortTile - 1) / kSortTile);
  size_t tbytes = carve_bytes<int32_t>(E) + 2 * carve_bytes<unsigned long long>(E) +
                  2 * carve_bytes<int32_t>(E) + carve_bytes<int32_t>(16 * ntiles) +
                  carve_bytes<int64_t>(16 * ntiles + 1) + carve_bytes<int64_t>(scan_tmp_elems(16 * ntiles)) +
                  carve_bytes<int32_t>(8) + 2 * carve_bytes<int32_t>(E) + 2 * carve_bytes<int64_t>(E + 1) +
                  carve_bytes<int64_t>(scan_tmp_elems(E)) + carve_bytes<unsigned long long>(E);
  BufferPtr tb;
  st = alloc_buffer(tbytes, s, &tb);
  if (st) return st;
  Carve ct{(char*)tb->ptr};
  int32_t* src = ct.take<int32_t>(E);
  unsigned long long* k0 = ct.take<unsigned long long>(E);
  unsigned long long* k1 = ct.take<unsigned long long>(E);
  int32_t* v0 = ct.take<int32_t>(E);
  int32_t* v1 = ct.take<int32_t>(E);
  int32_t* hist = ct.take<int32_t>(16 * ntiles);
  int64_t* hoff = ct.take<int64_t>(16 * ntiles + 1);
  int64_t* stmp = ct.take<int64_t>(scan_tmp_elems(16 * ntiles));
  int32_t* counts = ct.take<int32_t>(8);
  int32_t* segf = ct.take<int32_t>(E);
  int32_t* labf = ct.take<int32_t>(E);
  int64_t* segi = ct.take<int64_t>(E + 1);
  int64_t* labi = ct.take<int64_t>(E + 1);
  int64_t* etmp = ct.take<int64_t>(scan_tmp_elems(E));
  unsigned long long* vkeys = ct.take<unsigned long long>(E);
  int64_t lm_counts[2][2] = {{0, 0}, {0, 0}};
  FSTC_CUDA_TRY(cudaMemsetAsync(counts, 0, 8 * sizeof(int32_t), s));

  if (E > 0) {
    k_arc_src<<<nblk(E, 256), 256, 0, s>>>(V, E, h->row_ptr, src);
    FSTC_LAUNCH_CHECK();
  }
  const int NB = bits_for(V > 0 ? V - 1 : 0);
  for (int k = 0; k < 4; ++k) {
    const bool by_ol = (k == kOutByOlabel || k == kInByOlabel);
    const bool out = (k == kOutByOlabel || k == kOutByIlabel);
    const int32_t* label = by_ol ? h->olabel : h->ilabel;
    const int32_t* node = out ? src : h->dst;
    const int32_t* other = out ? h->dst : src;
    const int32_t* carry = by_ol ? h->ilabel : h->olabel;  // A role carries ilabel, B role olabel
    const int LB = bits_for((int64_t)(by_ol ? max_ol : max_il) + 1);
    const int bits = NB + LB;
    View& w = h->views[k];
    if (E > 0) {
      k_make_keys<<<nblk(E, 256), 256, 0, s>>>(E, node, label, LB, k0, v0);
      FSTC_LAUNCH_CHECK();
      unsigned long long* ka = k0;
      unsigned long long* kb = k1;
      int32_t* va = v0;
      int32_t* vbv = v1;
      for (int shift = 0; shift < bits; shift += 4) {
        k_radix_hist<<<(unsigned)ntiles, kSortThreads, 0, s>>>(ka, E, shift, hist, (int)ntiles);
        FSTC_LAUNCH_CHECK();
        st = exclusive_scan_i32(hist, 16 * ntiles, hoff, stmp, s);
        if (st) return st;
        k_radix_scatter<<<(unsigned)ntiles, kSortThreads, 0, s>>>(ka, va, E, shift, hoff, (int)ntiles, kb, vbv);
        FSTC_LAUNCH_CHECK();
        std::swap(ka, kb);
        std::swap(va, vbv);
      }
      k_gather_view<<<nblk(E, 256), 256, 0, s>>>(E, va, label, other, carry, h->weight, w.key, w.other, w.carry,
                                                 w.w, w.arc, w.cw);
      FSTC_LAUNCH_CHECK();
      k_view_offsets<<<nblk(E + 1, 256), 256, 0, s>>>(V, E, ka, LB, w.off);
      FSTC_LAUNCH_CHECK();
      k_view_items<<<nblk(std::max<int64_t>(E, V), 256), 256, 0, s>>>(V, E, w.off, w.key, w.other, ka, LB, w.cw,
                                                                        w.ikd, w.isrc, w.ikcw);
      FSTC_LAUNCH_CHECK();
      if (!by_ol) {  // B role: label-major segment index
        FSTC_CUDA_TRY(cudaMemcpyAsync(vkeys, ka, sizeof(unsigned long long) * E, cudaMemcpyDeviceToDevice, s));
        k_lm_keys<<<nblk(E, 256), 256, 0, s>>>(E, vkeys, LB, NB, w.key, k0, v0);
        FSTC_LAUNCH_CHECK();
        unsigned long long* la = k0;
        unsigned long long* lb = k1;
        int32_t* pa = v0;
        int32_t* pb = v1;
        for (int shift = 0; shift < bits; shift += 4) {
          k_radix_hist<<<(unsigned)ntiles, kSortThreads, 0, s>>>(la, E, shift, hist, (int)ntiles);
          FSTC_LAUNCH_CHECK();
          st = exclusive_scan_i32(hist, 16 * ntiles, hoff, stmp, s);
          if (st) return st;
          k_radix_scatter<<<(unsigned)ntiles, kSortThreads, 0, s>>>(la, pa, E, shift, hoff, (int)ntiles, lb, pb);
          FSTC_LAUNCH_CHECK();
          std::swap(la, lb);
          std::swap(pa, pb);
        }
        k_lm_flags<<<nblk(E, 256), 256, 0, s>>>(E, la, pa, NB, w.other, w.lm_other, w.lm_pos, segf, labf);
        FSTC_LAUNCH_CHECK();
        st = exclusive_scan_i32(segf, E, segi, etmp, s);
        if (st) return st;
        st = exclusive_scan_i32(labf, E, labi, etmp, s);
        if (st) return st;
        k_lm_scatter<<<nblk(E + 1, 256), 256, 0, s>>>(E, la, NB, segf, labf, segi, labi, w.seg_node, w.seg_beg,
                                                       w.lab_val, w.lab_seg);
        FSTC_LAUNCH_CHECK();
        const int slot = k == kOutByIlabel ? 0 : 1;
        FSTC_CUDA_TRY(cudaMemcpyAsync(&lm_counts[slot][0], segi + E, 8, cudaMemcpyDeviceToHost, s));
        FSTC_CUDA_TRY(cudaMemcpyAsync(&lm_counts[slot][1], labi + E, 8, cudaMemcpyDeviceToHost, s));
      }
      k_view_maxdeg<<<std::min(nblk(V, 256), 1184u), 256, 0, s>>>(V, w.off, counts + 2 + k);
      FSTC_LAUNCH_CHECK();
    } else {
      FSTC_CUDA_TRY(cudaMemsetAsync(w.off, 0, sizeof(int32_t) * (V + 1), s));
      if (V > 0) {
        k_view_items<<<nblk(V, 256), 256, 0, s>>>(V, 0, w.off, w.key, w.other, nullptr, LB, w.cw, w.ikd, w.isrc,
                                                  w.ikcw);
        FSTC_LAUNCH_CHECK();
      }
    }

  }
  if (V > 0) {
    k_flag_lists<<<1, 1024, 0, s>>>(V, h->is_start, h->is_accept, h->start_list, h->accept_list, counts);
    FSTC_LAUNCH_CHECK();
  }
  {
    int32_t hc[8];
    FSTC_CUDA_TRY(cudaMemcpyAsync(hc, counts, sizeof(hc), cudaMemcpyDeviceToHost, s));
    FSTC_CUDA_TRY(cudaStreamSynchronize(s));
    h->n_start = V > 0 ? hc[0] : 0;
    h->n_accept = V > 0 ? hc[1] : 0;
    h->max_ilabel = max_il;
    h->max_olabel = max_ol;
    for (int k = 0; k < 4; ++k) h->views[k].max_deg = E > 0 ? hc[2 + k] : 0;
    h->views[kOutByIlabel].nseg = (int32_t)lm_counts[0][0];
    h->views[kOutByIlabel].nlab = (int32_t)lm_counts[0][1];
    h->views[kInByIlabel].nseg = (int32_t)lm_counts[1][0];
    h->views[kInByIlabel].nlab = (int32_t)lm_counts[1][1];
  }
  tb.reset();  // stream-ordered free after the work above
  h->has_views = true;
  return FST_OK;
}

// Views for a composed handle used as a compose input (labels are already valid).
fst_status ensure_views(fst* h, cudaStream_t s) {
  if (h->has_views) return FST_OK;
  BufferPtr tb;
  fst_status st = alloc_buffer(4 * sizeof(int32_t), s, &tb);
  if (st) return st;
  int32_t* out = (int32_t*)tb->ptr;
  int32_t init[4] = {0, -1, -1, 0};
  FSTC_CUDA_TRY(cudaMemcpyAsync(out, init, sizeof(init), cudaMemcpyHostToDevice, s));
  if (h->E > 0) {
    k_validate_arcs<<<nblk(h->E, 256), 256, 0, s>>>(h->V, h->E, h->ilabel, h->olabel, h->dst, h->weight, out);
    FSTC_LAUNCH_CHECK();
  }
  int32_t res[4];
  FSTC_CUDA_TRY(cudaMemcpyAsync(res, out, sizeof(res), cudaMemcpyDeviceToHost, s));
  FSTC_CUDA_TRY(cudaStreamSynchronize(s));
  return build_views(h, s, res[1], res[2]);
}

}  // namespace fstc

using namespace fstc;

extern "C" fst_status fst_create(const fst_desc* d, void* stream, fst_handle* out) {
  if (!d || !out) {
    set_error(FST_E_INVALID_ARG, "fst_create: NULL argument");
    return FST_E_INVALID_ARG;
  }
  *out = nullptr;
  const int32_t V = d->num_states;
  const int64_t E = d->num_arcs;
  if (V < 0 || E < 0 || !d->row_ptr || (E > 0 && (!d->ilabel || !d->olabel || !d->dst || !d->weight)) ||
      (V > 0 && (!d->is_start || !d->is_accept)) || (d->memory != FST_MEM_DEVICE && d->memory != FST_MEM_HOST)) {
    set_error(FST_E_INVALID_ARG, "fst_create: bad descriptor (V=%d E=%lld)", V, (long long)E);
    return FST_E_INVALID_ARG;
  }
  if (V == INT32_MAX || E >= INT32_MAX) {
    set_error(FST_E_CAPACITY, "fst_create: V and E must be < 2^31");
    return FST_E_CAPACITY;
  }
  fst_status rd = device_ready();
  if (rd) return rd;
  cudaStream_t s = (cudaStream_t)stream;
  fst* h = new fst();
  h->V = V;
  h->E = E;
  h->stream = s;
  size_t bytes = carve_bytes<int64_t>(V + 1) + 3 * carve_bytes<int32_t>(E) + carve_bytes<float>(E) +
                 2 * carve_bytes<uint8_t>(V) + carve_bytes<int32_t>(4);
  BufferPtr b;
  fst_status st = alloc_buffer(bytes, s, &b);
  if (st) {
    delete h;
    return st;
  }
  h->buffers.push_back(b);
  Carve cv{(char*)b->ptr};
  h->row_ptr = cv.take<int64_t>(V + 1);
  h->ilabel = cv.take<int32_t>(E);
  h->olabel = cv.take<int32_t>(E);
  h->dst = cv.take<int32_t>(E);
  h->weight = cv.take<float>(E);
  h->is_start = cv.take<uint8_t>(V);
  h->is_accept = cv.take<uint8_t>(V);
  int32_t* vout = cv.take<int32_t>(4);
  const cudaMemcpyKind kind = d->memory == FST_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
#define CP(dst_, src_, n_)                                                                      \
  if ((n_) > 0) {                                                                               \
    cudaError_t _e = cudaMemcpyAsync(dst_, src_, (n_), kind, s);                                \
    if (_e != cudaSuccess) {                                                                    \
      set_error(FST_E_CUDA, "fst_create: upload failed: %s", cudaGetErrorString(_e));           \
      delete h;                                                                                 \
      return FST_E_CUDA;                                                                        \
    }                                                                                           \
  }
  CP(h->row_ptr, d->row_ptr, sizeof(int64_t) * (V + 1));
  CP(h->ilabel, d->ilabel, sizeof(int32_t) * E);
  CP(h->olabel, d->olabel, sizeof(int32_t) * E);
  CP(h->dst, d->dst, sizeof(int32_t) * E);
  CP(h->weight, d->weight, sizeof(float) * E);
  CP(h->is_start, d->is_start, V);
  CP(h->is_accept, d->is_accept, V);
#undef CP
  int32_t init[4] = {0, -1, -1, 0};
  cudaMemcpyAsync(vout, init, sizeof(init), cudaMemcpyHostToDevice, s);
  k_validate_states<<<nblk((int64_t)V + 1, 256), 256, 0, s>>>(V, E, h->row_ptr, h->is_start, h->is_accept, vout);
  count_launch();
  if (E > 0) {
    k_validate_arcs<<<nblk(E, 256), 256, 0, s>>>(V, E, h->ilabel, h->olabel, h->dst, h->weight, vout);
    count_launch();
  }
  int32_t res[4];
  cudaMemcpyAsync(res, vout, sizeof(res), cudaMemcpyDeviceToHost, s);
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) {
    set_error(FST_E_CUDA, "fst_create: %s", cudaGetErrorString(e));
    delete h;
    return FST_E_CUDA;
  }
  if (res[0] != 0) {
    set_error(FST_E_INVALID_GRAPH, "fst_create: invalid graph (%s%s%s%s%s%s%s)", res[0] & 1 ? "row_ptr[0]!=0 " : "",
              res[0] & 2 ? "row_ptr decreasing " : "", res[0] & 4 ? "row_ptr[V]!=E " : "",
              res[0] & 8 ? "dst out of range " : "", res[0] & 16 ? "label < -1 " : "",
              res[0] & 32 ? "non-finite weight " : "", res[0] & 64 ? "flag not 0/1" : "");
    delete h;
    return FST_E_INVALID_GRAPH;
  }
  st = build_views(h, s, res[1], res[2]);
  if (st) {
    delete h;
    return st;
  }
  *out = h;
  return FST_OK;
}
