/*
 * oracle/compose.c -- CPU oracle for eager trimmed WFST composition (arXiv 2110.02848).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (paper_2110_02848_b200/, include/)
 * may include, link or call this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it.  It shares no code with the CUDA path.
 *
 * What it computes (Algorithm 1 "Sequential Composition"), step by step in
 * the paper's order, with the epsilon moves of DESIGN.md reading N1:
 *   line 3      R <- co-accessible pairs: backward BFS from accept pairs "nearly identical ...
 *               but proceeds backwards from the accept states", using the exact
 *               reverse of the forward moves M1/M2/M3.
 *   lines 4-11  every start pair (s_a, s_b) in R becomes a start state (accept iff both accept).
 *   lines 12-31 FIFO loop: pop (u_a,u_b); (i) all arc pairs e_a x e_b with o_a == i_b (eps==eps
 *               is a literal match, M1); dst pair must be in R; create it if new; add arc
 *               i_a:o_b (reading 3: the paper's "o_a:i_b" is garbled) with weight w_a + w_b as ONE
 *               IEEE binary32 add (reading 12); (ii) M2: e_a with o_a = eps, B stays, arc i_a:eps
 *               weight w_a (bit copy); (iii) M3: e_b with i_b = eps, A stays, arc eps:o_b, w_b.
 * Data layout follows §3.2: per-arc SoA arrays plus in/out adjacency with
 * offsets; in-adjacency is stable by arc index (the Fig. 1 example).
 *
 * Provenance (the autodiff use of the composed graph): every
 * arc also records the arc pair (e_a, e_b) that produced it (-1 for the side that stays).
 *
 * Pins (tests/test_oracle.py): Fig. 1 arrays, hand fixtures F1-F5, brute-force Eq. (1) path
 * scores on tiny DAGs, Delannoy path counts with eps, plain-definition trim(P_N1), identity and
 * trellis special cases.  Build: gcc -O2 -std=c99 (no -ffast-math: no FTZ/DAZ, SSE float adds).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_EPS (-1)

typedef struct {
  int32_t V;
  int64_t E;
  const int64_t* row_ptr; /* [V+1] arcs grouped by source */
  const int32_t* ilabel;
  const int32_t* olabel;
  const int32_t* dst;
  const float* weight;
  const uint8_t* is_start;
  const uint8_t* is_accept;
} orc_fst;

typedef struct {
  int32_t V;
  int64_t E;
  int64_t* row_ptr;
  int32_t* ilabel;
  int32_t* olabel;
  int32_t* dst;
  float* weight;
  uint8_t* is_start;
  uint8_t* is_accept;
  int32_t* pair_a;
  int32_t* pair_b;
  int32_t* level; /* BFS level of each state (FIFO discovery distance), for Fig. 2 profiles */
  int32_t* arc_a; /* provenance: the arc pair (e_a, e_b) of Alg. 1 line 13 that */
  int32_t* arc_b; /* produced each arc; -1 = that side stays (M3 for arc_a, M2 for arc_b) */
  int32_t* pair_f; /* eps-filter state of each state (orc_compose_filtered only; NULL otherwise) */
} orc_graph;

/* ---------------------------------------------------------------- adjacency (§3.2) */
typedef struct {
  int32_t* src;     /* [E] "input node indices" */
  int64_t* in_off;  /* [V+1] inArcOffset */
  int64_t* in_arcs; /* [E] inArcs, consecutive by node, ascending arc index within a node */
} orc_adj;

static int adj_build(const orc_fst* g, orc_adj* a) {
  int64_t E = g->E, e;
  int32_t V = g->V, v;
  a->src = (int32_t*)malloc(sizeof(int32_t) * (size_t)(E ? E : 1));
  a->in_off = (int64_t*)calloc((size_t)V + 1, sizeof(int64_t));
  a->in_arcs = (int64_t*)malloc(sizeof(int64_t) * (size_t)(E ? E : 1));
  if (!a->src || !a->in_off || !a->in_arcs) return -1;
  for (v = 0; v < V; ++v)
    for (e = g->row_ptr[v]; e < g->row_ptr[v + 1]; ++e) a->src[e] = v;
  for (e = 0; e < E; ++e) a->in_off[g->dst[e] + 1]++;
  for (v = 0; v < V; ++v) a->in_off[v + 1] += a->in_off[v];
  {
    int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * ((size_t)V + 1));
    if (!cur) return -1;
    memcpy(cur, a->in_off, sizeof(int64_t) * ((size_t)V + 1));
    for (e = 0; e < E; ++e) a->in_arcs[cur[g->dst[e]]++] = e;
    free(cur);
  }
  return 0;
}

static void adj_free(orc_adj* a) {
  free(a->src);
  free(a->in_off);
  free(a->in_arcs);
}

/* exported for the Fig. 1 golden test: inArcOffset / inArcs of one FST */
int orc_in_adjacency(const orc_fst* g, int64_t* in_off, int64_t* in_arcs) {
  orc_adj a;
  if (adj_build(g, &a)) return -1;
  memcpy(in_off, a.in_off, sizeof(int64_t) * ((size_t)g->V + 1));
  if (g->E) memcpy(in_arcs, a.in_arcs, sizeof(int64_t) * (size_t)g->E);
  adj_free(&a);
  return 0;
}

/* ---------------------------------------------------------------- line 3: co-accessible set R */
/* R[(v_a * V_B) + v_b] = 1 iff the pair can reach an accept pair by forward moves; computed by a
 * backward FIFO BFS from all accept pairs over the reversed moves. */
static int coaccessible(const orc_fst* A, const orc_fst* B, const orc_adj* aA, const orc_adj* aB,
                        uint8_t* R) {
  int64_t VB = B->V, P = (int64_t)A->V * B->V;
  int64_t* Q = (int64_t*)malloc(sizeof(int64_t) * (size_t)(P ? P : 1));
  int64_t head = 0, tail = 0;
  int32_t fa, fb;
  if (!Q) return -1;
  memset(R, 0, (size_t)P);
  for (fa = 0; fa < A->V; ++fa) {
    if (!A->is_accept[fa]) continue;
    for (fb = 0; fb < B->V; ++fb) {
      if (!B->is_accept[fb]) continue;
      R[fa * VB + fb] = 1;
      Q[tail++] = fa * VB + fb;
    }
  }
  while (head < tail) {
    int64_t v = Q[head++];
    int32_t va = (int32_t)(v / VB), vb = (int32_t)(v % VB);
    int64_t i, j;
    /* reversed M1: in-arc pairs with o_a == i_b; predecessor (src e_a, src e_b) */
    for (i = aA->in_off[va]; i < aA->in_off[va + 1]; ++i) {
      int64_t ea = aA->in_arcs[i];
      for (j = aB->in_off[vb]; j < aB->in_off[vb + 1]; ++j) {
        int64_t eb = aB->in_arcs[j];
        int64_t p;
        if (A->olabel[ea] != B->ilabel[eb]) continue;
        p = (int64_t)aA->src[ea] * VB + aB->src[eb];
        if (!R[p]) { R[p] = 1; Q[tail++] = p; }
      }
    }
    /* reversed M2: A in-arc with o_a = eps; B stays */
    for (i = aA->in_off[va]; i < aA->in_off[va + 1]; ++i) {
      int64_t ea = aA->in_arcs[i], p;
      if (A->olabel[ea] != ORC_EPS) continue;
      p = (int64_t)aA->src[ea] * VB + vb;
      if (!R[p]) { R[p] = 1; Q[tail++] = p; }
    }
    /* reversed M3: B in-arc with i_b = eps; A stays */
    for (j = aB->in_off[vb]; j < aB->in_off[vb + 1]; ++j) {
      int64_t eb = aB->in_arcs[j], p;
      if (B->ilabel[eb] != ORC_EPS) continue;
      p = (int64_t)va * VB + aB->src[eb];
      if (!R[p]) { R[p] = 1; Q[tail++] = p; }
    }
  }
  free(Q);
  return 0;
}

int orc_coaccessible(const orc_fst* A, const orc_fst* B, uint8_t* R) {
  orc_adj aA, aB;
  int rc;
  if (adj_build(A, &aA) || adj_build(B, &aB)) return -1;
  rc = coaccessible(A, B, &aA, &aB, R);
  adj_free(&aA);
  adj_free(&aB);
  return rc;
}

/* ---------------------------------------------------------------- growable output */
typedef struct {
  int64_t n, cap;
  int32_t *il, *ol, *dst, *aa, *ab;
  float* w;
  uint64_t* dig;  /* digest mode (orc_digest): arcs are hashed into dig[0..1] instead of stored */
} arcbuf;

/* ---------------------------------------------------------------- order-independent digest
 * SURVEY 8(d) d.7, for parity at sizes where the composed graph is too large to compare array by
 * array: D_f = sum over states s of hS_f(key(s), start, accept, out-degree) + sum over arcs of
 * hA_f(key(src), key(dst), ilabel, olabel, weight bits), mod 2^64, f = 0, 1 (two seeds).  Sums of
 * per-state / per-arc hashes are invariant under state renumbering and arc order, so equal canonical
 * graphs (reading 24) have equal digests.  fin = the splitmix64 finalizer. */
static uint64_t fin(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static const uint64_t kDigestSeed[2] = {0x9E3779B97F4A7C15ull, 0xD1B54A32D192ED03ull};
static uint64_t hash_state(int f, uint64_t key, int st, int ac, uint64_t deg) {
  return fin(fin(fin(key ^ kDigestSeed[f]) ^ (uint64_t)(st | (ac << 1) | 4)) ^ deg);
}
static uint64_t hash_arc(int f, uint64_t ksrc, uint64_t kdst, int32_t il, int32_t ol, float w) {
  uint32_t wb;
  memcpy(&wb, &w, 4);
  return fin(fin(fin(fin(ksrc ^ kDigestSeed[f] ^ 0x5555555555555555ull) ^ kdst) ^
                 (((uint64_t)(uint32_t)il << 32) | (uint32_t)ol)) ^ wb);
}

static int arc_push(arcbuf* b, int32_t il, int32_t ol, int32_t d, float w, int32_t aa, int32_t ab,
                    uint64_t ksrc, uint64_t kdst) {
  if (b->dig) {
    b->dig[0] += hash_arc(0, ksrc, kdst, il, ol, w);
    b->dig[1] += hash_arc(1, ksrc, kdst, il, ol, w);
    b->n++;
    return 0;
  }
  if (b->n == b->cap) {
    int64_t nc = b->cap ? 2 * b->cap : 1024;
    int32_t* a1 = (int32_t*)realloc(b->il, sizeof(int32_t) * (size_t)nc);
    int32_t* a2;
    int32_t* a3;
    float* a4;
    if (!a1) return -1;
    b->il = a1;
    a2 = (int32_t*)realloc(b->ol, sizeof(int32_t) * (size_t)nc);
    if (!a2) return -1;
    b->ol = a2;
    a3 = (int32_t*)realloc(b->dst, sizeof(int32_t) * (size_t)nc);
    if (!a3) return -1;
    b->dst = a3;
    a4 = (float*)realloc(b->w, sizeof(float) * (size_t)nc);
    if (!a4) return -1;
    b->w = a4;
    a1 = (int32_t*)realloc(b->aa, sizeof(int32_t) * (size_t)nc);
    if (!a1) return -1;
    b->aa = a1;
    a1 = (int32_t*)realloc(b->ab, sizeof(int32_t) * (size_t)nc);
    if (!a1) return -1;
    b->ab = a1;
    b->cap = nc;
  }
  b->il[b->n] = il;
  b->ol[b->n] = ol;
  b->dst[b->n] = d;
  b->w[b->n] = w;
  b->aa[b->n] = aa;
  b->ab[b->n] = ab;
  b->n++;
  return 0;
}

/* ---------------------------------------------------------------- Algorithm 1 */
void orc_free(orc_graph* g) {
  if (!g) return;
  free(g->row_ptr); free(g->ilabel); free(g->olabel); free(g->dst); free(g->weight);
  free(g->is_start); free(g->is_accept); free(g->pair_a); free(g->pair_b); free(g->level);
  free(g->arc_a); free(g->arc_b); free(g->pair_f);
  memset(g, 0, sizeof(*g));
}

static int compose_impl(const orc_fst* A, const orc_fst* B, orc_graph* C, uint64_t* dig) {
  int64_t VB = B->V, P = (int64_t)A->V * B->V;
  orc_adj aA, aB;
  uint8_t* R;
  int32_t* id;          /* V_A x V_B state-index table: -1 = "not in C" */
  int32_t *pa = NULL, *pb = NULL, *lv = NULL;
  uint8_t *st = NULL, *ac = NULL;
  int64_t* rp = NULL;
  int64_t ns = 0, capS = 0, u, i;
  arcbuf arcs;
  int32_t sa, sb;
  memset(C, 0, sizeof(*C));
  memset(&arcs, 0, sizeof(arcs));
  arcs.dig = dig;
  if (adj_build(A, &aA) || adj_build(B, &aB)) return -1;
  /* line 2-3 */
  R = (uint8_t*)malloc((size_t)(P ? P : 1));
  id = (int32_t*)malloc(sizeof(int32_t) * (size_t)(P ? P : 1));
  if (!R || !id) return -1;
  if (coaccessible(A, B, &aA, &aB, R)) return -1;
  for (i = 0; i < P; ++i) id[i] = -1;

#define NEW_STATE(va_, vb_, lev_)                                                         \
  do {                                                                                    \
    if (ns == capS) {                                                                     \
      capS = capS ? 2 * capS : 1024;                                                      \
      pa = (int32_t*)realloc(pa, sizeof(int32_t) * (size_t)capS);                        \
      pb = (int32_t*)realloc(pb, sizeof(int32_t) * (size_t)capS);                        \
      lv = (int32_t*)realloc(lv, sizeof(int32_t) * (size_t)capS);                        \
      st = (uint8_t*)realloc(st, (size_t)capS);                                          \
      ac = (uint8_t*)realloc(ac, (size_t)capS);                                          \
      rp = (int64_t*)realloc(rp, sizeof(int64_t) * (size_t)(capS + 1));                  \
      if (!pa || !pb || !lv || !st || !ac || !rp) return -1;                             \
    }                                                                                     \
    id[(int64_t)(va_) * VB + (vb_)] = (int32_t)ns;                                        \
    pa[ns] = (va_); pb[ns] = (vb_); lv[ns] = (lev_); st[ns] = 0;                          \
    ac[ns] = (uint8_t)(A->is_accept[(va_)] && B->is_accept[(vb_)]);                      \
    ns++;                                                                                 \
  } while (0)

  /* lines 4-11: start pairs in R become start states (and enter Q) */
  for (sa = 0; sa < A->V; ++sa) {
    if (!A->is_start[sa]) continue;
    for (sb = 0; sb < B->V; ++sb) {
      if (!B->is_start[sb]) continue;
      if (!R[(int64_t)sa * VB + sb]) continue;
      NEW_STATE(sa, sb, 0);
      st[ns - 1] = 1;
    }
  }
  /* lines 12-31: FIFO over Q.  States enter Q in creation order, so Q's head is state id u. */
  for (u = 0; u < ns; ++u) {
    int32_t ua = pa[u], ub = pb[u];
    int64_t ea, eb;
    rp[u] = arcs.n;
    /* (i) M1: all arc pairs leaving u_a and u_b (line 13), in arc order */
    for (ea = A->row_ptr[ua]; ea < A->row_ptr[ua + 1]; ++ea) {
      for (eb = B->row_ptr[ub]; eb < B->row_ptr[ub + 1]; ++eb) {
        int32_t oa = A->olabel[ea], ib = B->ilabel[eb], va, vb;
        int64_t v;
        float w;
        if (oa != ib) continue;                    /* lines 16-18 */
        va = A->dst[ea]; vb = B->dst[eb];          /* line 19 */
        v = (int64_t)va * VB + vb;
        if (!R[v]) continue;                       /* lines 20-22 */
        if (id[v] < 0) NEW_STATE(va, vb, lv[u] + 1); /* lines 23-28 */
        w = A->weight[ea] + B->weight[eb];         /* line 29-30: one binary32 add */
        if (arc_push(&arcs, A->ilabel[ea], B->olabel[eb], id[v], w, (int32_t)ea, (int32_t)eb,
                     (uint64_t)ua * VB + ub, (uint64_t)v)) return -1;
      }
    }
    /* (ii) M2: e_a with o_a = eps, B stays */
    for (ea = A->row_ptr[ua]; ea < A->row_ptr[ua + 1]; ++ea) {
      int32_t va;
      int64_t v;
      if (A->olabel[ea] != ORC_EPS) continue;
      va = A->dst[ea];
      v = (int64_t)va * VB + ub;
      if (!R[v]) continue;
      if (id[v] < 0) NEW_STATE(va, ub, lv[u] + 1);
      if (arc_push(&arcs, A->ilabel[ea], ORC_EPS, id[v], A->weight[ea], (int32_t)ea, -1, (uint64_t)ua * VB + ub,
                   (uint64_t)v)) return -1;
    }
    /* (iii) M3: e_b with i_b = eps, A stays */
    for (eb = B->row_ptr[ub]; eb < B->row_ptr[ub + 1]; ++eb) {
      int32_t vb;
      int64_t v;
      if (B->ilabel[eb] != ORC_EPS) continue;
      vb = B->dst[eb];
      v = (int64_t)ua * VB + vb;
      if (!R[v]) continue;
      if (id[v] < 0) NEW_STATE(ua, vb, lv[u] + 1);
      if (arc_push(&arcs, ORC_EPS, B->olabel[eb], id[v], B->weight[eb], -1, (int32_t)eb, (uint64_t)ua * VB + ub,
                   (uint64_t)v)) return -1;
    }
    if (dig) {  /* the state's own term: its key, flags and out-degree (its arcs were just pushed) */
      const uint64_t deg = (uint64_t)(arcs.n - rp[u]);
      dig[0] += hash_state(0, (uint64_t)ua * VB + ub, st[u], ac[u], deg);
      dig[1] += hash_state(1, (uint64_t)ua * VB + ub, st[u], ac[u], deg);
    }
  }
#undef NEW_STATE
  if (!rp) rp = (int64_t*)malloc(sizeof(int64_t));
  rp[ns] = arcs.n;
  C->V = (int32_t)ns;
  C->E = arcs.n;
  C->row_ptr = rp;
  C->ilabel = arcs.il;
  C->olabel = arcs.ol;
  C->dst = arcs.dst;
  C->weight = arcs.w;
  C->arc_a = arcs.aa;
  C->arc_b = arcs.ab;
  C->is_start = st;
  C->is_accept = ac;
  C->pair_a = pa;
  C->pair_b = pb;
  C->level = lv;
  free(R);
  free(id);
  adj_free(&aA);
  adj_free(&aB);
  return 0;
}

int orc_compose(const orc_fst* A, const orc_fst* B, orc_graph* C) { return compose_impl(A, B, C, NULL); }

/* Algorithm 1 with the composed arcs streamed into the digest (nothing stored per arc): out[0] = V_C,
 * out[1] = E_C, out[2..3] = D_0, D_1.  Memory is the pair tables only, so configs[3] at full size fits. */
int orc_digest(const orc_fst* A, const orc_fst* B, uint64_t* out) {
  orc_graph C;
  uint64_t dig[2] = {0, 0};
  int rc = compose_impl(A, B, &C, dig);
  if (rc) return rc;
  out[0] = (uint64_t)C.V;
  out[1] = (uint64_t)C.E;
  out[2] = dig[0];
  out[3] = dig[1];
  orc_free(&C);
  return 0;
}

/* ---------------------------------------------------------------- eps-filtered variant */
/* The paper claims eps support but gives no redundancy filter; without one,
 * interleaved eps moves duplicate paths (the Delannoy inflation of reading N1).  This is the standard
 * three-state eps filter as SPEC.md states it (S:150-153 FilterState, S:168-177 match_moves), run
 * through Algorithm 1's structure over triples (u_a, u_b, f), f in
 * {0 = MATCH, 1 = A_EPS, 2 = B_EPS}:
 *   (1) MATCH     e_a x e_b, o_a == i_b != eps, from any f          -> (dst e_a, dst e_b, 0), w_a + w_b
 *   (2) EPS-BOTH  e_a x e_b, o_a == i_b == eps, only from f = 0      -> (dst e_a, dst e_b, 0), w_a + w_b
 *   (3) EPS-A     e_a with o_a = eps, B stays, from f in {0, 1}      -> (dst e_a, u_b, 1),     w_a
 *   (4) EPS-B     e_b with i_b = eps, A stays, from f in {0, 2}      -> (u_a, dst e_b, 2),     w_b
 * Start triples (s_a, s_b, 0); accept triples (f_a, f_b, any f).  R (line 3) is computed exactly on
 * the triple space by the reversed moves (SPEC's unfiltered R + final trim sweep gives the same
 * trim graph).  Labels, weights and provenance as in orc_compose. */
#define FK(a_, b_, f_) ((((int64_t)(a_)) * VB + (b_)) * 3 + (f_))

static int coaccessible_filtered(const orc_fst* A, const orc_fst* B, const orc_adj* aA, const orc_adj* aB,
                                 uint8_t* R) {
  int64_t VB = B->V, P3 = (int64_t)A->V * B->V * 3;
  int64_t* Q = (int64_t*)malloc(sizeof(int64_t) * (size_t)(P3 ? P3 : 1));
  int64_t head = 0, tail = 0;
  int32_t fa, fb, f;
  if (!Q) return -1;
  memset(R, 0, (size_t)P3);
#define MARK(p_) do { int64_t q_ = (p_); if (!R[q_]) { R[q_] = 1; Q[tail++] = q_; } } while (0)
  for (fa = 0; fa < A->V; ++fa) {
    if (!A->is_accept[fa]) continue;
    for (fb = 0; fb < B->V; ++fb)
      if (B->is_accept[fb])
        for (f = 0; f < 3; ++f) MARK(FK(fa, fb, f));
  }
  while (head < tail) {
    int64_t v = Q[head++];
    int32_t vf = (int32_t)(v % 3), va = (int32_t)(v / 3 / VB), vb = (int32_t)(v / 3 % VB);
    int64_t i, j;
    if (vf == 0) { /* reversed (1) from any f, reversed (2) from f = 0 */
      for (i = aA->in_off[va]; i < aA->in_off[va + 1]; ++i) {
        int64_t ea = aA->in_arcs[i];
        for (j = aB->in_off[vb]; j < aB->in_off[vb + 1]; ++j) {
          int64_t eb = aB->in_arcs[j];
          if (A->olabel[ea] != B->ilabel[eb]) continue;
          if (A->olabel[ea] != ORC_EPS) {
            for (f = 0; f < 3; ++f) MARK(FK(aA->src[ea], aB->src[eb], f));
          } else {
            MARK(FK(aA->src[ea], aB->src[eb], 0));
          }
        }
      }
    } else if (vf == 1) { /* reversed (3): from f in {0, 1} */
      for (i = aA->in_off[va]; i < aA->in_off[va + 1]; ++i) {
        int64_t ea = aA->in_arcs[i];
        if (A->olabel[ea] != ORC_EPS) continue;
        MARK(FK(aA->src[ea], vb, 0));
        MARK(FK(aA->src[ea], vb, 1));
      }
    } else { /* reversed (4): from f in {0, 2} */
      for (j = aB->in_off[vb]; j < aB->in_off[vb + 1]; ++j) {
        int64_t eb = aB->in_arcs[j];
        if (B->ilabel[eb] != ORC_EPS) continue;
        MARK(FK(va, aB->src[eb], 0));
        MARK(FK(va, aB->src[eb], 2));
      }
    }
  }
#undef MARK
  free(Q);
  return 0;
}

int orc_compose_filtered(const orc_fst* A, const orc_fst* B, orc_graph* C) {
  int64_t VB = B->V, P3 = (int64_t)A->V * B->V * 3;
  orc_adj aA, aB;
  uint8_t* R;
  int32_t* id; /* V_A x V_B x 3 state-index table */
  int32_t *pa = NULL, *pb = NULL, *pf = NULL, *lv = NULL;
  uint8_t *st = NULL, *ac = NULL;
  int64_t* rp = NULL;
  int64_t ns = 0, capS = 0, u, i;
  arcbuf arcs;
  int32_t sa, sb;
  memset(C, 0, sizeof(*C));
  memset(&arcs, 0, sizeof(arcs));
  if (adj_build(A, &aA) || adj_build(B, &aB)) return -1;
  R = (uint8_t*)malloc((size_t)(P3 ? P3 : 1));
  id = (int32_t*)malloc(sizeof(int32_t) * (size_t)(P3 ? P3 : 1));
  if (!R || !id) return -1;
  if (coaccessible_filtered(A, B, &aA, &aB, R)) return -1;
  for (i = 0; i < P3; ++i) id[i] = -1;

#define NEW_STATE3(va_, vb_, vf_, lev_)                                                   \
  do {                                                                                    \
    if (ns == capS) {                                                                     \
      capS = capS ? 2 * capS : 1024;                                                      \
      pa = (int32_t*)realloc(pa, sizeof(int32_t) * (size_t)capS);                        \
      pb = (int32_t*)realloc(pb, sizeof(int32_t) * (size_t)capS);                        \
      pf = (int32_t*)realloc(pf, sizeof(int32_t) * (size_t)capS);                        \
      lv = (int32_t*)realloc(lv, sizeof(int32_t) * (size_t)capS);                        \
      st = (uint8_t*)realloc(st, (size_t)capS);                                          \
      ac = (uint8_t*)realloc(ac, (size_t)capS);                                          \
      rp = (int64_t*)realloc(rp, sizeof(int64_t) * (size_t)(capS + 1));                  \
      if (!pa || !pb || !pf || !lv || !st || !ac || !rp) return -1;                      \
    }                                                                                     \
    id[FK(va_, vb_, vf_)] = (int32_t)ns;                                                  \
    pa[ns] = (va_); pb[ns] = (vb_); pf[ns] = (vf_); lv[ns] = (lev_); st[ns] = 0;         \
    ac[ns] = (uint8_t)(A->is_accept[(va_)] && B->is_accept[(vb_)]);                      \
    ns++;                                                                                 \
  } while (0)
#define ADD_MOVE(va_, vb_, vf_, il_, ol_, w_, xa_, xb_)                                   \
  do {                                                                                    \
    int64_t v_ = FK(va_, vb_, vf_);                                                       \
    if (R[v_]) {                                                                          \
      if (id[v_] < 0) NEW_STATE3(va_, vb_, vf_, lv[u] + 1);                               \
      if (arc_push(&arcs, il_, ol_, id[v_], w_, xa_, xb_, 0, 0)) return -1;               \
    }                                                                                     \
  } while (0)

  /* lines 4-11: start triples (s_a, s_b, MATCH) in R */
  for (sa = 0; sa < A->V; ++sa) {
    if (!A->is_start[sa]) continue;
    for (sb = 0; sb < B->V; ++sb) {
      if (!B->is_start[sb] || !R[FK(sa, sb, 0)]) continue;
      NEW_STATE3(sa, sb, 0, 0);
      st[ns - 1] = 1;
    }
  }
  /* lines 12-31 */
  for (u = 0; u < ns; ++u) {
    int32_t ua = pa[u], ub = pb[u], uf = pf[u];
    int64_t ea, eb;
    rp[u] = arcs.n;
    /* (1) MATCH and (2) EPS-BOTH: arc pairs in arc order */
    for (ea = A->row_ptr[ua]; ea < A->row_ptr[ua + 1]; ++ea) {
      for (eb = B->row_ptr[ub]; eb < B->row_ptr[ub + 1]; ++eb) {
        int32_t oa = A->olabel[ea];
        float w;
        if (oa != B->ilabel[eb]) continue;
        if (oa == ORC_EPS && uf != 0) continue; /* EPS-BOTH only from MATCH */
        w = A->weight[ea] + B->weight[eb];      /* one binary32 add */
        ADD_MOVE(A->dst[ea], B->dst[eb], 0, A->ilabel[ea], B->olabel[eb], w, (int32_t)ea, (int32_t)eb);
      }
    }
    /* (3) EPS-A from f in {MATCH, A_EPS} */
    if (uf != 2)
      for (ea = A->row_ptr[ua]; ea < A->row_ptr[ua + 1]; ++ea)
        if (A->olabel[ea] == ORC_EPS)
          ADD_MOVE(A->dst[ea], ub, 1, A->ilabel[ea], ORC_EPS, A->weight[ea], (int32_t)ea, -1);
    /* (4) EPS-B from f in {MATCH, B_EPS} */
    if (uf != 1)
      for (eb = B->row_ptr[ub]; eb < B->row_ptr[ub + 1]; ++eb)
        if (B->ilabel[eb] == ORC_EPS)
          ADD_MOVE(ua, B->dst[eb], 2, ORC_EPS, B->olabel[eb], B->weight[eb], -1, (int32_t)eb);
  }
#undef ADD_MOVE
#undef NEW_STATE3
  if (!rp) rp = (int64_t*)malloc(sizeof(int64_t));
  rp[ns] = arcs.n;
  C->V = (int32_t)ns;
  C->E = arcs.n;
  C->row_ptr = rp;
  C->ilabel = arcs.il;
  C->olabel = arcs.ol;
  C->dst = arcs.dst;
  C->weight = arcs.w;
  C->arc_a = arcs.aa;
  C->arc_b = arcs.ab;
  C->is_start = st;
  C->is_accept = ac;
  C->pair_a = pa;
  C->pair_b = pb;
  C->pair_f = pf;
  C->level = lv;
  free(R);
  free(id);
  adj_free(&aA);
  adj_free(&aB);
  return 0;
}
#undef FK

/* ---------------------------------------------------------------- canonical form (reading 24) */
/* States renumbered by ascending key(a,b) = a*V_B + b; arcs of a row sorted by
 * (dst key, ilabel, olabel, weight bits as uint32). */
static const int64_t* g_keys;
static int cmp_state(const void* x, const void* y) {
  int64_t a = g_keys[*(const int32_t*)x], b = g_keys[*(const int32_t*)y];
  return (a > b) - (a < b);
}
typedef struct {
  int32_t dst, il, ol;
  uint32_t wbits;
  float w;
  int32_t aa, ab;
} carc;
static int cmp_arc(const void* x, const void* y) {
  const carc* a = (const carc*)x;
  const carc* b = (const carc*)y;
  if (a->dst != b->dst) return a->dst < b->dst ? -1 : 1;
  if (a->il != b->il) return a->il < b->il ? -1 : 1;
  if (a->ol != b->ol) return a->ol < b->ol ? -1 : 1;
  if (a->wbits != b->wbits) return a->wbits < b->wbits ? -1 : 1;
  if (a->aa != b->aa) return a->aa < b->aa ? -1 : 1; /* provenance breaks ties between identical arcs */
  if (a->ab != b->ab) return a->ab < b->ab ? -1 : 1;
  return 0;
}

int orc_canonicalize(orc_graph* C, int32_t VB) {
  int32_t V = C->V, s;
  int64_t E = C->E, k = 0;
  int64_t* keys = (int64_t*)malloc(sizeof(int64_t) * (size_t)(V ? V : 1));
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(V ? V : 1));
  int32_t* newid = (int32_t*)malloc(sizeof(int32_t) * (size_t)(V ? V : 1));
  orc_graph D;
  carc* tmp = NULL;
  int64_t tcap = 0;
  if (!keys || !order || !newid) return -1;
  for (s = 0; s < V; ++s) {
    keys[s] = (int64_t)C->pair_a[s] * VB + C->pair_b[s];
    if (C->pair_f) keys[s] = keys[s] * 3 + C->pair_f[s]; /* SPEC PairState key (a*V_B + b)*3 + f */
    order[s] = s;
  }
  g_keys = keys;
  qsort(order, (size_t)V, sizeof(int32_t), cmp_state);
  for (s = 0; s < V; ++s) newid[order[s]] = s;
  memset(&D, 0, sizeof(D));
  D.V = V; D.E = E;
  D.row_ptr = (int64_t*)malloc(sizeof(int64_t) * ((size_t)V + 1));
  D.ilabel = (int32_t*)malloc(sizeof(int32_t) * (size_t)(E ? E : 1));
  D.olabel = (int32_t*)malloc(sizeof(int32_t) * (size_t)(E ? E : 1));
  D.dst = (int32_t*)malloc(sizeof(int32_t) * (size_t)(E ? E : 1));
  D.weight = (float*)malloc(sizeof(float) * (size_t)(E ? E : 1));
  D.is_start = (uint8_t*)malloc((size_t)(V ? V : 1));
  D.is_accept = (uint8_t*)malloc((size_t)(V ? V : 1));
  D.pair_a = (int32_t*)malloc(sizeof(int32_t) * (size_t)(V ? V : 1));
  D.pair_b = (int32_t*)malloc(sizeof(int32_t) * (size_t)(V ? V : 1));
  D.level = (int32_t*)malloc(sizeof(int32_t) * (size_t)(V ? V : 1));
  D.arc_a = (int32_t*)malloc(sizeof(int32_t) * (size_t)(E ? E : 1));
  D.arc_b = (int32_t*)malloc(sizeof(int32_t) * (size_t)(E ? E : 1));
  if (C->pair_f) D.pair_f = (int32_t*)malloc(sizeof(int32_t) * (size_t)(V ? V : 1));
  for (s = 0; s < V; ++s) {
    int32_t o = order[s];
    int64_t lo = C->row_ptr[o], hi = C->row_ptr[o + 1], n = hi - lo, e;
    D.row_ptr[s] = k;
    D.is_start[s] = C->is_start[o];
    D.is_accept[s] = C->is_accept[o];
    D.pair_a[s] = C->pair_a[o];
    D.pair_b[s] = C->pair_b[o];
    D.level[s] = C->level[o];
    if (C->pair_f) D.pair_f[s] = C->pair_f[o];
    if (n > tcap) {
      tcap = n;
      tmp = (carc*)realloc(tmp, sizeof(carc) * (size_t)tcap);
      if (!tmp) return -1;
    }
    for (e = 0; e < n; ++e) {
      carc* c = &tmp[e];
      c->dst = newid[C->dst[lo + e]];
      c->il = C->ilabel[lo + e];
      c->ol = C->olabel[lo + e];
      c->w = C->weight[lo + e];
      memcpy(&c->wbits, &c->w, 4);
      c->aa = C->arc_a[lo + e];
      c->ab = C->arc_b[lo + e];
    }
    qsort(tmp, (size_t)n, sizeof(carc), cmp_arc);
    for (e = 0; e < n; ++e) {
      D.dst[k] = tmp[e].dst;
      D.ilabel[k] = tmp[e].il;
      D.olabel[k] = tmp[e].ol;
      D.weight[k] = tmp[e].w;
      D.arc_a[k] = tmp[e].aa;
      D.arc_b[k] = tmp[e].ab;
      k++;
    }
  }
  D.row_ptr[V] = k;
  free(tmp);
  free(keys);
  free(order);
  free(newid);
  orc_free(C);
  *C = D;
  return 0;
}
