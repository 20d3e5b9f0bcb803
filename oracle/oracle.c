/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for Recurrent Arc
 * Consistency (RAC), arXiv 2407.11388.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code with the CUDA path (paper_2407_11388_b200/csrc): no
 * headers, helpers or tables; the only common dependency is the seeded input
 * generator synth/csp_synth.h, which holds none of the method's arithmetic.
 *
 * Layout (deliberately different from the GPU's [x][a][y] masks): a per-arc
 * adjacency list.  For variable x, nbr[x][k] is the k-th constrained
 * neighbour y (ascending), and sup[x][k*dom[x] + a] is the support set
 * c_xy|(x,a) = { tau[y] | tau in rel(c_xy), tau[x] = a }
 * as a bitset over dom(y).  C_x is { c_{x,nbr[x][k]} }.
 * Domain states are one uint64 per variable, bit a set iff (x,a) in D.
 *
 * Functions:
 *   orc_rac     -- O1: the RAC recurrence, Eq. 1 run
 *                  literally and synchronously, with Alg. 1's loop and checks
 *                  (lines 198-210).  Counts iterations, records removal epochs.
 *   orc_ac3     -- O2: textbook AC-3 (propagation queue + revision, PAPER.md
 *                  line 29; SPEC.md ac3_engine lines 262-310), FIFO.
 *   orc_is_ac   -- the definition of arc consistency.
 *   orc_certify -- O4: D_out = D_ac certificate: arc-consistency audit plus
 *                  Lemma 1 (proof 304-308) applied to
 *                  every removal in epoch order.
 *   orc_row_supported_synth -- one (x,a) support test against D computed
 *                  straight from the generator (sampled checks at any size).
 *
 * O3 (brute-force union of all arc-consistent subsets)
 * is in oracle/__init__.py (pure Python, tiny instances).
 *
 * Readings of the paper:
 *   R1  Eq. 1 is read in the intersection form of line 59: (x,a) is removed
 *       at step k iff some declared c_xy in C_x has c_xy|(x,a) ∩ D_{k-1}(y) = ∅.
 *   R2  "∃y" ranges over declared constraints only; absent pairs never remove.
 *   R3  iterations = number of passes executed, including the final no-change
 *       pass; on wipeout the detecting pass is counted (Alg. 1 loop body count).
 *   R4  update is synchronous (Jacobi): step k reads only D_{k-1}.
 *   R5  wipeout is checked before convergence (Alg. 1).
 *   R6  on wipeout (stop mode) the output is D after the detecting pass.
 *   R7  an empty row in D_in: one pass runs, then WIPEOUT (iterations = 1).
 *   FULL mode ignores wipeouts and iterates to the definitional D_ac.
 *
 * Parity pins: see tests/test_oracle.py (brute force, closed forms, hand
 * traces, AC-3 agreement, certificate, invariants).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../synth/csp_synth.h"

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_WIPEOUT 1
#define ORC_EINVAL (-1)

typedef struct {
  int n;
  int *dom;        /* dom[x], 1..64                                  */
  int *deg;        /* number of constrained neighbours of x          */
  int **nbr;       /* nbr[x][k] ascending                            */
  int **rev;       /* rev[x][k] = index of x in nbr[nbr[x][k]]       */
  uint64_t **sup;  /* sup[x][k*dom[x] + a] = c_{x,nbr[x][k]}|(x,a)   */
} orc_csp;

static uint64_t dom_mask(int k) { return k >= 64 ? ~0ULL : ((1ULL << k) - 1ULL); }

static int popc64(uint64_t v) {
  int c = 0;
  while (v) { v &= v - 1; ++c; }
  return c;
}

void orc_free(orc_csp *c) {
  if (!c) return;
  for (int x = 0; x < c->n; ++x) {
    if (c->nbr) free(c->nbr[x]);
    if (c->rev) free(c->rev[x]);
    if (c->sup) free(c->sup[x]);
  }
  free(c->nbr); free(c->rev); free(c->sup); free(c->deg); free(c->dom);
  free(c);
}

static orc_csp *alloc_csp(int n, const int *dom) {
  orc_csp *c = (orc_csp *)calloc(1, sizeof(orc_csp));
  if (!c) return NULL;
  c->n = n;
  c->dom = (int *)calloc((size_t)n, sizeof(int));
  c->deg = (int *)calloc((size_t)n, sizeof(int));
  c->nbr = (int **)calloc((size_t)n, sizeof(int *));
  c->rev = (int **)calloc((size_t)n, sizeof(int *));
  c->sup = (uint64_t **)calloc((size_t)n, sizeof(uint64_t *));
  if (!c->dom || !c->deg || !c->nbr || !c->rev || !c->sup) { orc_free(c); return NULL; }
  for (int x = 0; x < n; ++x) c->dom[x] = dom[x];
  return c;
}

/* Index of y in nbr[x] (ascending), or -1. */
static int arc_index(const orc_csp *c, int x, int y) {
  int lo = 0, hi = c->deg[x] - 1;
  while (lo <= hi) {
    int mid = (lo + hi) / 2;
    if (c->nbr[x][mid] == y) return mid;
    if (c->nbr[x][mid] < y) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

/* After deg[] is known: allocate per-x arrays. */
static int alloc_arcs(orc_csp *c) {
  for (int x = 0; x < c->n; ++x) {
    size_t k = (size_t)(c->deg[x] > 0 ? c->deg[x] : 1);
    c->nbr[x] = (int *)malloc(k * sizeof(int));
    c->rev[x] = (int *)malloc(k * sizeof(int));
    c->sup[x] = (uint64_t *)calloc(k * (size_t)c->dom[x], sizeof(uint64_t));
    if (!c->nbr[x] || !c->rev[x] || !c->sup[x]) return -1;
  }
  return 0;
}

static void fill_rev(orc_csp *c) {
  for (int x = 0; x < c->n; ++x)
    for (int k = 0; k < c->deg[x]; ++k) c->rev[x][k] = arc_index(c, c->nbr[x][k], x);
}

static int cmp_int(const void *a, const void *b) {
  int u = *(const int *)a, v = *(const int *)b;
  return (u > v) - (u < v);
}

/*
 * Build from explicit relations: constraint r is on (xs[r], ys[r]) and
 * rows[r*row_stride + a] is row a of rel(c_{xs[r],ys[r]}) (bit b set iff
 * (a,b) allowed).  Either orientation is accepted.  Returns NULL on invalid
 * input (x == y, out of range, a duplicate unordered pair, bits beyond the
 * domain sizes).
 */
orc_csp *orc_build(int n, const int *dom, int n_rel, const int *xs, const int *ys,
                   const uint64_t *rows, int row_stride) {
  if (n < 1) return NULL;
  for (int x = 0; x < n; ++x)
    if (dom[x] < 1 || dom[x] > 64) return NULL;
  orc_csp *c = alloc_csp(n, dom);
  if (!c) return NULL;
  for (int r = 0; r < n_rel; ++r) {
    int x = xs[r], y = ys[r];
    if (x < 0 || y < 0 || x >= n || y >= n || x == y) { orc_free(c); return NULL; }
    c->deg[x]++; c->deg[y]++;
  }
  if (alloc_arcs(c)) { orc_free(c); return NULL; }
  int *fill = (int *)calloc((size_t)n, sizeof(int));
  for (int r = 0; r < n_rel; ++r) {
    c->nbr[xs[r]][fill[xs[r]]++] = ys[r];
    c->nbr[ys[r]][fill[ys[r]]++] = xs[r];
  }
  free(fill);
  for (int x = 0; x < n; ++x) {
    qsort(c->nbr[x], (size_t)c->deg[x], sizeof(int), cmp_int);
    for (int k = 1; k < c->deg[x]; ++k)
      if (c->nbr[x][k] == c->nbr[x][k - 1]) { orc_free(c); return NULL; } /* duplicate pair */
  }
  for (int r = 0; r < n_rel; ++r) {
    int x = xs[r], y = ys[r];
    int kx = arc_index(c, x, y), ky = arc_index(c, y, x);
    for (int a = 0; a < dom[x]; ++a) {
      uint64_t row = rows[(size_t)r * (size_t)row_stride + (size_t)a];
      if (row & ~dom_mask(dom[y])) { orc_free(c); return NULL; }
      /* arc x -> y: c_xy|(x,a) is row a itself */
      c->sup[x][(size_t)kx * dom[x] + a] = row;
      /* arc y -> x: c_yx|(y,b) = { a : (a,b) allowed } -- the transpose */
      for (int b = 0; b < dom[y]; ++b)
        if ((row >> b) & 1ULL) c->sup[y][(size_t)ky * dom[y] + b] |= 1ULL << a;
    }
    for (int a = dom[x]; a < row_stride; ++a)
      if (rows[(size_t)r * (size_t)row_stride + (size_t)a]) { orc_free(c); return NULL; }
  }
  fill_rev(c);
  return c;
}

/* Build the seeded random instance of synth/csp_synth.h (uniform domain d). */
orc_csp *orc_build_synth(int n, int d, uint64_t dens_q32, uint32_t t_q16, uint64_t seed) {
  if (n < 1 || d < 1 || d > 64) return NULL;
  int *dom = (int *)malloc((size_t)n * sizeof(int));
  for (int x = 0; x < n; ++x) dom[x] = d;
  orc_csp *c = alloc_csp(n, dom);
  free(dom);
  if (!c) return NULL;
  /* pass 1: degrees */
  for (int x = 0; x < n; ++x)
    for (int y = x + 1; y < n; ++y)
      if (synth_present(seed, (uint32_t)n, (uint32_t)x, (uint32_t)y, dens_q32)) { c->deg[x]++; c->deg[y]++; }
  if (alloc_arcs(c)) { orc_free(c); return NULL; }
  /* pass 2: neighbour lists, ascending in y */
  int *fill = (int *)calloc((size_t)n, sizeof(int));
  for (int x = 0; x < n; ++x)
    for (int y = 0; y < n; ++y) {
      if (y == x) continue;
      int lo = x < y ? x : y, hi = x < y ? y : x;
      if (synth_present(seed, (uint32_t)n, (uint32_t)lo, (uint32_t)hi, dens_q32)) c->nbr[x][fill[x]++] = y;
    }
  free(fill);
  for (int x = 0; x < n; ++x) {
    for (int k = 0; k < c->deg[x]; ++k) {
      int y = c->nbr[x][k];
      if (x < y) {
        for (int a = 0; a < d; ++a)
          c->sup[x][(size_t)k * d + a] =
              synth_row(seed, (uint32_t)n, (uint32_t)d, (uint32_t)x, (uint32_t)y, (uint32_t)a, t_q16);
      } else {
        /* c_xy with x > y is the transpose of c_yx: (a,b) allowed in c_xy iff (b,a) allowed in c_yx */
        for (int b = 0; b < d; ++b) {
          uint64_t row_b = synth_row(seed, (uint32_t)n, (uint32_t)d, (uint32_t)y, (uint32_t)x, (uint32_t)b, t_q16);
          for (int a = 0; a < d; ++a)
            if ((row_b >> a) & 1ULL) c->sup[x][(size_t)k * d + a] |= 1ULL << b;
        }
      }
    }
  }
  fill_rev(c);
  return c;
}

/*
 * Partial build for sampled CPU timing at sizes the full oracle instance does
 * not fit (C4): arcs only for variables x in [x_lo, x_hi) (all their
 * neighbours y), other variables get no arcs.  Only orc_pass_block may be used
 * on it.
 */
orc_csp *orc_build_synth_block(int n, int d, uint64_t dens_q32, uint32_t t_q16, uint64_t seed, int x_lo, int x_hi) {
  if (n < 1 || d < 1 || d > 64 || x_lo < 0 || x_hi > n || x_lo > x_hi) return NULL;
  int *dom = (int *)malloc((size_t)n * sizeof(int));
  for (int x = 0; x < n; ++x) dom[x] = d;
  orc_csp *c = alloc_csp(n, dom);
  free(dom);
  if (!c) return NULL;
  for (int x = x_lo; x < x_hi; ++x)
    for (int y = 0; y < n; ++y) {
      if (y == x) continue;
      int lo = x < y ? x : y, hi = x < y ? y : x;
      if (synth_present(seed, (uint32_t)n, (uint32_t)lo, (uint32_t)hi, dens_q32)) c->deg[x]++;
    }
  if (alloc_arcs(c)) { orc_free(c); return NULL; }
  for (int x = x_lo; x < x_hi; ++x) {
    int k = 0;
    for (int y = 0; y < n; ++y) {
      if (y == x) continue;
      int lo = x < y ? x : y, hi = x < y ? y : x;
      if (!synth_present(seed, (uint32_t)n, (uint32_t)lo, (uint32_t)hi, dens_q32)) continue;
      c->nbr[x][k] = y;
      if (x < y) {
        for (int a = 0; a < d; ++a)
          c->sup[x][(size_t)k * d + a] =
              synth_row(seed, (uint32_t)n, (uint32_t)d, (uint32_t)x, (uint32_t)y, (uint32_t)a, t_q16);
      } else {
        for (int b = 0; b < d; ++b) {
          uint64_t row_b = synth_row(seed, (uint32_t)n, (uint32_t)d, (uint32_t)y, (uint32_t)x, (uint32_t)b, t_q16);
          for (int a = 0; a < d; ++a)
            if ((row_b >> a) & 1ULL) c->sup[x][(size_t)k * d + a] |= 1ULL << b;
        }
      }
      ++k;
    }
  }
  return c;
}

/*
 * One step of Eq. 1 restricted to the rows of variables [x_lo, x_hi):
 * out[x - x_lo] = { a ∈ D(x) : ∀ c_xy ∈ C_x  c_xy|(x,a) ∩ D(y) ≠ ∅ }.
 * Same loop as orc_rac's step.  Returns the number of values removed.
 */
int64_t orc_pass_block(const orc_csp *c, const uint64_t *D, int x_lo, int x_hi, uint64_t *out) {
  int64_t removed = 0;
  for (int x = x_lo; x < x_hi; ++x) {
    uint64_t nx = D[x];
    for (int a = 0; a < c->dom[x]; ++a) {
      if (!((D[x] >> a) & 1ULL)) continue;
      for (int kk = 0; kk < c->deg[x]; ++kk) {
        int y = c->nbr[x][kk];
        if ((c->sup[x][(size_t)kk * c->dom[x] + a] & D[y]) == 0) { nx &= ~(1ULL << a); ++removed; break; }
      }
    }
    out[x - x_lo] = nx;
  }
  return removed;
}

int orc_n(const orc_csp *c) { return c->n; }
int orc_degree(const orc_csp *c, int x) { return c->deg[x]; }

/* c_xy|(x,a) as a bitset over dom(y); *present = 0 (and result 0) if no c_xy. */
uint64_t orc_support(const orc_csp *c, int x, int y, int a, int *present) {
  int k = (x == y) ? -1 : arc_index(c, x, y);
  if (k < 0) { *present = 0; return 0; }
  *present = 1;
  return c->sup[x][(size_t)k * c->dom[x] + a];
}

/*
 * The definition of arc consistency:
 *   D is AC  <=>  for all (x,a) in D, for all c_xy in C_x: c_xy|(x,a) ∩ D(y) ≠ ∅.
 * Returns 1 if D is arc consistent, else 0.
 */
int orc_is_ac(const orc_csp *c, const uint64_t *D) {
  for (int x = 0; x < c->n; ++x)
    for (int a = 0; a < c->dom[x]; ++a) {
      if (!((D[x] >> a) & 1ULL)) continue;
      for (int k = 0; k < c->deg[x]; ++k) {
        int y = c->nbr[x][k];
        if ((c->sup[x][(size_t)k * c->dom[x] + a] & D[y]) == 0) return 0;
      }
    }
  return 1;
}

/*
 * O1: the RAC recurrence, Eq. 1, run literally.
 *
 *   D^(0)_~ac = ∅;  D^(k)_~ac = D^(k-1)_~ac ∪ {(x,a) | ∃ c_xy ∈ C_x: c_xy|(x,a) ⊆ D^(k-1)_~ac}
 *
 * in the complement form D_k = D_in \ D^(k)_~ac with the intersection test of
 * line 59 (reading R1): (x,a) ∈ D_{k-1} is removed at step k iff some declared
 * c_xy has c_xy|(x,a) ∩ D_{k-1}(y) = ∅.  Step k reads only D_{k-1} (R4): the
 * result goes into a fresh array.  Loop control follows Alg. 1 tensorAC (lines
 * 198-210): after each pass, wipeout is checked first (line 203, R5), then
 * "nothing changed" ends the loop (line 200/206; Prop. 1 end condition,
 * line 125).  iterations counts every pass executed (R3).
 *
 * removed_at (nullable, n*64 int32): removed_at[x*64+a] = k if (x,a) was
 * removed at step k, 0 otherwise (the per-step sets V^(k) of Prop. 2).
 * full != 0: do not stop at a wipeout; iterate to the fixpoint (the
 * definitional D_ac, in which a wiped component is emptied).
 * Returns ORC_OK or ORC_WIPEOUT.
 */
int orc_rac(const orc_csp *c, const uint64_t *d_in, uint64_t *d_out, int *iterations,
            int32_t *removed_at, int full) {
  int n = c->n;
  uint64_t *prev = (uint64_t *)calloc((size_t)n, sizeof(uint64_t));
  uint64_t *next = (uint64_t *)calloc((size_t)n, sizeof(uint64_t));
  memcpy(prev, d_in, (size_t)n * sizeof(uint64_t));
  if (removed_at) memset(removed_at, 0, (size_t)n * 64 * sizeof(int32_t));
  int k = 0, status = ORC_OK;
  for (;;) {
    ++k;
    /* one step of Eq. 1: every test reads prev (= D_{k-1}) only */
    for (int x = 0; x < n; ++x) {
      next[x] = prev[x];
      for (int a = 0; a < c->dom[x]; ++a) {
        if (!((prev[x] >> a) & 1ULL)) continue;
        for (int kk = 0; kk < c->deg[x]; ++kk) {
          int y = c->nbr[x][kk];
          uint64_t s = c->sup[x][(size_t)kk * c->dom[x] + a]; /* c_xy|(x,a) */
          if ((s & prev[y]) == 0) {                            /* ∩ D_{k-1}(y) = ∅ */
            next[x] &= ~(1ULL << a);
            if (removed_at) removed_at[x * 64 + a] = k;
            break;
          }
        }
      }
    }
    int wipe = 0, changed = 0;
    for (int x = 0; x < n; ++x) {
      if (next[x] == 0) wipe = 1;
      if (next[x] != prev[x]) changed = 1;
    }
    memcpy(prev, next, (size_t)n * sizeof(uint64_t));
    if (wipe && !full) { status = ORC_WIPEOUT; break; } /* Alg. 1 */
    if (!changed) { status = wipe ? ORC_WIPEOUT : ORC_OK; break; }
  }
  memcpy(d_out, prev, (size_t)n * sizeof(uint64_t));
  *iterations = k;
  free(prev); free(next);
  return status;
}

/*
 * O1 on `threads` host threads (0 = all), for the CPU baseline timed on every
 * core of the host: the same synchronous step as orc_rac -- every variable's
 * new word depends only on prev -- with the variables of a step split over
 * OpenMP threads, then the same wipeout-first / convergence checks.  No removal
 * epochs.  Results equal orc_rac for every thread count (tests/test_oracle.py).
 */
int orc_rac_par(const orc_csp *c, const uint64_t *d_in, uint64_t *d_out, int *iterations, int full, int threads) {
  int n = c->n;
  uint64_t *prev = (uint64_t *)calloc((size_t)n, sizeof(uint64_t));
  uint64_t *next = (uint64_t *)calloc((size_t)n, sizeof(uint64_t));
  if (!prev || !next) { free(prev); free(next); return ORC_EINVAL; }
  memcpy(prev, d_in, (size_t)n * sizeof(uint64_t));
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#endif
  int k = 0, status = ORC_OK;
  for (;;) {
    ++k;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 16)
#endif
    for (int x = 0; x < n; ++x) {
      uint64_t nx = prev[x];
      for (int a = 0; a < c->dom[x]; ++a) {
        if (!((prev[x] >> a) & 1ULL)) continue;
        for (int kk = 0; kk < c->deg[x]; ++kk) {
          int y = c->nbr[x][kk];
          if ((c->sup[x][(size_t)kk * c->dom[x] + a] & prev[y]) == 0) { nx &= ~(1ULL << a); break; }
        }
      }
      next[x] = nx;
    }
    int wipe = 0, changed = 0;
    for (int x = 0; x < n; ++x) {
      if (next[x] == 0) wipe = 1;
      if (next[x] != prev[x]) changed = 1;
    }
    memcpy(prev, next, (size_t)n * sizeof(uint64_t));
    if (wipe && !full) { status = ORC_WIPEOUT; break; }
    if (!changed) { status = wipe ? ORC_WIPEOUT : ORC_OK; break; }
  }
  memcpy(d_out, prev, (size_t)n * sizeof(uint64_t));
  *iterations = k;
  free(prev); free(next);
  return status;
}

/* O1 on S independent states (the batched workload), states spread over
 * `threads` OpenMP threads (0 = all); state s at d_in + s*n.  No epochs. */
int orc_rac_many(const orc_csp *c, int S, const uint64_t *d_in, uint64_t *d_out, int *iterations, int *status,
                 int full, int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
  for (int s = 0; s < S; ++s)
    status[s] = orc_rac(c, d_in + (size_t)s * c->n, d_out + (size_t)s * c->n, iterations + s, NULL, full);
  return 0;
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/*
 * O5: Alg. 1 tensorAC(Vars, @changed) as written:
 *   while |@changed| != 0:
 *     Vars = tensorRevise(Vars, @changed)   -- (x,a) kept iff for every y in
 *         @changed (with a declared c_xy, reading R2) c_xy|(x,a) ∩ D(y) ≠ ∅
 *     if some #Vals == 0: inconsistency      -- checked first (R5)
 *     @changed = { x : #Vals(x) != #Vals_pre(x) }
 * seeds = the initial @changed (P:392 calls it with [idx] after an
 * assignment; the root call P:381 passes all variables).  An empty seed list
 * runs no pass (iterations = 0).  Same outputs as orc_rac.
 */
int orc_rac_seeded(const orc_csp *c, const uint64_t *d_in, const int32_t *seeds, int n_seeds, uint64_t *d_out,
                   int *iterations, int32_t *removed_at, int full) {
  int n = c->n;
  uint64_t *prev = (uint64_t *)calloc((size_t)n, sizeof(uint64_t));
  uint64_t *next = (uint64_t *)calloc((size_t)n, sizeof(uint64_t));
  char *chg = (char *)calloc((size_t)n, 1);
  memcpy(prev, d_in, (size_t)n * sizeof(uint64_t));
  if (removed_at) memset(removed_at, 0, (size_t)n * 64 * sizeof(int32_t));
  int n_chg = 0;
  for (int i = 0; i < n_seeds; ++i)
    if (seeds[i] >= 0 && seeds[i] < n && !chg[seeds[i]]) { chg[seeds[i]] = 1; ++n_chg; }
  int k = 0, status = ORC_OK;
  while (n_chg != 0) {
    ++k;
    for (int x = 0; x < n; ++x) {
      next[x] = prev[x];
      for (int a = 0; a < c->dom[x]; ++a) {
        if (!((prev[x] >> a) & 1ULL)) continue;
        for (int kk = 0; kk < c->deg[x]; ++kk) {
          int y = c->nbr[x][kk];
          if (!chg[y]) continue; /* Cons[*, @changed] only */
          if ((c->sup[x][(size_t)kk * c->dom[x] + a] & prev[y]) == 0) {
            next[x] &= ~(1ULL << a);
            if (removed_at) removed_at[x * 64 + a] = k;
            break;
          }
        }
      }
    }
    int wipe = 0;
    n_chg = 0;
    for (int x = 0; x < n; ++x) {
      if (next[x] == 0) wipe = 1;
      chg[x] = next[x] != prev[x];
      n_chg += chg[x];
    }
    memcpy(prev, next, (size_t)n * sizeof(uint64_t));
    if (wipe && !full) { status = ORC_WIPEOUT; break; }
    if (n_chg == 0 && wipe) status = ORC_WIPEOUT;
  }
  if (k == 0) {
    for (int x = 0; x < n; ++x)
      if (prev[x] == 0) status = ORC_WIPEOUT;
  }
  memcpy(d_out, prev, (size_t)n * sizeof(uint64_t));
  *iterations = k;
  free(prev); free(next); free(chg);
  return status;
}

/*
 * O6: Alg. 2 backtracking search, written
 * recursively: dfs(level, Vars) picks idx = heuristics() -- the unassigned
 * variable with the fewest values, lowest index on ties (the
 * paper leaves it open, line 389) -- and for each Val in Var[idx].nonzero()
 * (ascending) assigns it on a COPY of the parent's domains (the paper's
 * pseudocode reuses Vars across siblings, lines 390-393, reading R13) and
 * enforces.  engine 0: O5 tensorAC(Vars, [idx]) (line 392); 1: O1 full
 * recurrence; 2: O2 AC-3.  stats[0] assignments,
 * [1] sum of iterations (engine 2: of AC-3 revisions), [2] wipeouts, [3] solutions, [4] max depth,
 * [5] root iterations.  Returns 0 solution found (first one in solution[]),
 * 1 unsatisfiable, 2 budget exhausted.  all != 0: explore the whole tree.
 */
int orc_ac3(const orc_csp *c, const uint64_t *d_in, uint64_t *d_out, int64_t *revisions);

typedef struct {
  const orc_csp *c;
  int64_t budget;
  int engine, all, full;
  int64_t *stats;
  int32_t *solution;
  char *assigned;
  int found, out_of_budget;
} orc_search_ctx;

static int orc_enforce_engine(orc_search_ctx *s, const uint64_t *din, uint64_t *dout, int seed, int *iters) {
  if (s->engine == 0) return orc_rac_seeded(s->c, din, &seed, 1, dout, iters, NULL, s->full);
  if (s->engine == 1) return orc_rac(s->c, din, dout, iters, NULL, s->full);
  int64_t rev = 0;
  int st = orc_ac3(s->c, din, dout, &rev);
  *iters = (int)rev; /* engine 2 sums AC-3 revisions (Table 1's #Revision) */
  return st;
}

static int orc_dfs(orc_search_ctx *s, const uint64_t *D, int level) {
  const orc_csp *c = s->c;
  int n = c->n;
  int idx = -1, best = 65;
  for (int x = 0; x < n; ++x)
    if (!s->assigned[x] && popc64(D[x]) < best) { best = popc64(D[x]); idx = x; }
  s->assigned[idx] = 1;
  uint64_t *child = (uint64_t *)malloc((size_t)n * sizeof(uint64_t));
  uint64_t *out = (uint64_t *)malloc((size_t)n * sizeof(uint64_t));
  int stop = 0;
  for (int v = 0; v < 64 && !stop; ++v) {
    if (!((D[idx] >> v) & 1ULL)) continue;
    if (s->budget > 0 && s->stats[0] >= s->budget) { s->out_of_budget = 1; stop = 1; break; }
    memcpy(child, D, (size_t)n * sizeof(uint64_t));
    child[idx] = 1ULL << v; /* assign, lines 410-416 */
    int it = 0;
    int st = orc_enforce_engine(s, child, out, idx, &it);
    s->stats[0]++;
    s->stats[1] += it;
    if (st == ORC_WIPEOUT) { s->stats[2]++; continue; }
    if (level + 1 > s->stats[4]) s->stats[4] = level + 1;
    if (level + 1 == n) {
      s->stats[3]++;
      if (!s->found && s->solution)
        for (int x = 0; x < n; ++x)
          for (int b = 0; b < 64; ++b)
            if ((out[x] >> b) & 1ULL) { s->solution[x] = b; break; }
      s->found = 1;
      if (!s->all) stop = 1;
      continue;
    }
    if (orc_dfs(s, out, level + 1)) stop = 1;
  }
  free(child); free(out);
  s->assigned[idx] = 0;
  return stop;
}

int orc_search(const orc_csp *c, const uint64_t *d_in, int64_t max_assignments, int engine, int all, int full,
               int32_t *solution, int64_t *stats) {
  int n = c->n;
  for (int k = 0; k < 6; ++k) stats[k] = 0;
  uint64_t *root = (uint64_t *)malloc((size_t)n * sizeof(uint64_t));
  int it = 0, st;
  if (engine == 2) { int64_t rev; st = orc_ac3(c, d_in, root, &rev); }
  else st = orc_rac(c, d_in, root, &it, NULL, full);
  stats[5] = it;
  if (st == ORC_WIPEOUT) { free(root); return 1; }
  orc_search_ctx s = {c, max_assignments, engine, all, full, stats, solution, NULL, 0, 0};
  s.assigned = (char *)calloc((size_t)n, 1);
  orc_dfs(&s, root, 0);
  free(s.assigned);
  free(root);
  if (s.out_of_budget) return 2;
  return s.found ? 0 : 1;
}

/*
 * O2: AC-3 ("a propagation queue and a revision process";
 * SPEC.md ac3_engine lines 283-299).  FIFO queue of directed arcs (x,y),
 * initially every arc in ascending (x, y) order; revise(x,y) removes every
 * a ∈ D(x) with c_xy|(x,a) ∩ D(y) = ∅; if D(x) shrank, enqueue (z,x) for every
 * neighbour z ≠ y not already queued.  Plus an upfront empty-domain check
 * (without it, an empty isolated domain would be reported consistent).
 * Independent of O1 in algorithm, order and update discipline.
 * *revisions counts dequeues.  Returns ORC_OK (d_out = D_ac) or ORC_WIPEOUT.
 */
int orc_ac3(const orc_csp *c, const uint64_t *d_in, uint64_t *d_out, int64_t *revisions) {
  int n = c->n;
  memcpy(d_out, d_in, (size_t)n * sizeof(uint64_t));
  *revisions = 0;
  for (int x = 0; x < n; ++x)
    if (d_out[x] == 0) return ORC_WIPEOUT;
  size_t n_arcs = 0;
  size_t *off = (size_t *)malloc(((size_t)n + 1) * sizeof(size_t));
  for (int x = 0; x < n; ++x) { off[x] = n_arcs; n_arcs += (size_t)c->deg[x]; }
  off[n] = n_arcs;
  size_t cap = n_arcs + 1;
  int *qx = (int *)malloc(cap * sizeof(int));
  int *qk = (int *)malloc(cap * sizeof(int));
  char *inq = (char *)calloc(n_arcs + 1, 1);
  size_t head = 0, count = 0;
  for (int x = 0; x < n; ++x)
    for (int k = 0; k < c->deg[x]; ++k) {
      qx[(head + count) % cap] = x; qk[(head + count) % cap] = k; ++count;
      inq[off[x] + (size_t)k] = 1;
    }
  int status = ORC_OK;
  while (count) {
    int x = qx[head], k = qk[head];
    head = (head + 1) % cap; --count;
    inq[off[x] + (size_t)k] = 0;
    ++*revisions;
    int y = c->nbr[x][k];
    uint64_t before = d_out[x];
    for (int a = 0; a < c->dom[x]; ++a) {
      if (!((d_out[x] >> a) & 1ULL)) continue;
      if ((c->sup[x][(size_t)k * c->dom[x] + a] & d_out[y]) == 0) d_out[x] &= ~(1ULL << a);
    }
    if (d_out[x] != before) {
      if (d_out[x] == 0) { status = ORC_WIPEOUT; break; }
      for (int j = 0; j < c->deg[x]; ++j) {
        int z = c->nbr[x][j];
        if (z == y) continue;
        int kz = c->rev[x][j]; /* arc (z, x) */
        if (!inq[off[z] + (size_t)kz]) {
          inq[off[z] + (size_t)kz] = 1;
          qx[(head + count) % cap] = z; qk[(head + count) % cap] = kz; ++count;
        }
      }
    }
  }
  free(off); free(qx); free(qk); free(inq);
  return status;
}

/*
 * O4: certificate that d_out is exactly D_ac(d_in) (or, for a stop-mode
 * wipeout, that every removal is sound).
 *   (i)  [check_ac] d_out is arc consistent (definition, lines 49-61)
 *        => d_out ⊆ D_ac (D_ac is the union of all AC subsets, lines 62-63);
 *   (ii) every removed (x,a) with epoch t has a declared c_xy such that every
 *        b ∈ c_xy|(x,a) ∩ d_in(y) was removed at an epoch < t.  By induction
 *        on t with Lemma 1 (lines 79-82) every removed value is in D~ac
 *        => d_in \ d_out ⊆ D~ac.
 *   (i)+(ii) give d_out = D_ac.  Also checks d_out ⊆ d_in and that epochs are
 *   set exactly on removed values.
 * Returns 0 = accepted; 1 = not AC; 2 = d_out ⊄ d_in; 3 = bad epoch marks;
 * 4 = a removal without a Lemma-1 justification.
 */
int orc_certify(const orc_csp *c, const uint64_t *d_in, const uint64_t *d_out,
                const int32_t *removed_at, int check_ac) {
  int n = c->n;
  for (int x = 0; x < n; ++x)
    if (d_out[x] & ~d_in[x]) return 2;
  for (int x = 0; x < n; ++x)
    for (int a = 0; a < 64; ++a) {
      int in = (int)((d_in[x] >> a) & 1ULL), out = (int)((d_out[x] >> a) & 1ULL);
      int32_t t = removed_at[x * 64 + a];
      if (in && !out) { if (t < 1) return 3; }
      else if (t != 0) return 3;
    }
  if (check_ac && !orc_is_ac(c, d_out)) return 1;
  for (int x = 0; x < n; ++x)
    for (int a = 0; a < c->dom[x]; ++a) {
      if (!((d_in[x] >> a) & 1ULL) || ((d_out[x] >> a) & 1ULL)) continue;
      int32_t t = removed_at[x * 64 + a];
      int justified = 0;
      for (int k = 0; k < c->deg[x] && !justified; ++k) {
        int y = c->nbr[x][k];
        uint64_t s = c->sup[x][(size_t)k * c->dom[x] + a] & d_in[y];
        int all_earlier = 1;
        for (int b = 0; b < 64; ++b) {
          if (!((s >> b) & 1ULL)) continue;
          int32_t tb = ((d_out[y] >> b) & 1ULL) ? 0 : removed_at[y * 64 + b];
          if (tb < 1 || tb >= t) { all_earlier = 0; break; }
        }
        if (all_earlier) justified = 1;
      }
      if (!justified) return 4;
    }
  return 0;
}

/*
 * One support test computed straight from the generator (no instance build):
 * is (x,a) supported on every declared c_xy in C_x against D?  i.e. would
 * (x,a) ∈ D survive one step of Eq. 1 from D.  Used for sampled parity at
 * sizes where building the oracle's instance is too large (C4).
 * Returns 1 supported, 0 removed.
 */
int orc_row_supported_synth(int n, int d, uint64_t dens_q32, uint32_t t_q16, uint64_t seed,
                            int x, int a, const uint64_t *D) {
  for (int y = 0; y < n; ++y) {
    if (y == x) continue;
    int lo = x < y ? x : y, hi = x < y ? y : x;
    if (!synth_present(seed, (uint32_t)n, (uint32_t)lo, (uint32_t)hi, dens_q32)) continue;
    uint64_t s = 0; /* c_xy|(x,a) */
    if (x < y) {
      s = synth_row(seed, (uint32_t)n, (uint32_t)d, (uint32_t)x, (uint32_t)y, (uint32_t)a, t_q16);
    } else {
      for (int b = 0; b < d; ++b)
        if (synth_allowed(seed, (uint32_t)n, (uint32_t)d, (uint32_t)y, (uint32_t)x, (uint32_t)b, (uint32_t)a, t_q16))
          s |= 1ULL << b;
    }
    if ((s & D[y]) == 0) return 0;
  }
  return 1;
}


/* ======================================================================== */
/*
 * Wide domains (d > 64, up to 256 values).
 *
 * The same recurrence, Eq. 1 with Alg. 1's loop
 * (lines 198-210) and readings R1-R7, on domains wider than one machine word.
 * The paper fixes no domain-size limit (its Cons is a dense [n,d,n,d] fp32
 * tensor); only the bitset width changes here.  A domain state is
 * wq = ceil(dmax/64) uint64 words per variable: bit a of variable x is bit
 * (a % 64) of word D[x*wq + a/64].  Support sets c_xy|(x,a) are wq-word
 * bitsets over dom(y).  removed_at has n * 64*wq entries, (x,a) at x*64*wq + a.
 * Kept separate from the one-word functions above so that those stay exactly
 * as pinned; the pins of these (tests/test_oracle.py "wide"): value
 * duplication of a pinned one-word instance, the arc-consistency audit, the
 * Lemma-1 certificate and AC-3 agreement (orc_wac3).
 */
typedef struct {
  int n, wq;
  int *dom;
  int *deg;
  int **nbr;       /* ascending */
  uint64_t **sup;  /* sup[x][((size_t)k*dom[x] + a)*wq + w] */
} orc_wcsp;

void orc_wfree(orc_wcsp *c) {
  if (!c) return;
  for (int x = 0; x < c->n; ++x) {
    if (c->nbr) free(c->nbr[x]);
    if (c->sup) free(c->sup[x]);
  }
  free(c->nbr); free(c->sup); free(c->dom); free(c->deg);
  free(c);
}

static int wbit(const uint64_t *v, int b) { return (int)((v[b >> 6] >> (b & 63)) & 1ULL); }
static void wset(uint64_t *v, int b) { v[b >> 6] |= 1ULL << (b & 63); }

static orc_wcsp *walloc(int n, const int *dom) {
  int dmax = 1;
  for (int x = 0; x < n; ++x) if (dom[x] > dmax) dmax = dom[x];
  orc_wcsp *c = (orc_wcsp *)calloc(1, sizeof(orc_wcsp));
  if (!c) return NULL;
  c->n = n;
  c->wq = (dmax + 63) / 64;
  c->dom = (int *)calloc((size_t)n, sizeof(int));
  c->deg = (int *)calloc((size_t)n, sizeof(int));
  c->nbr = (int **)calloc((size_t)n, sizeof(int *));
  c->sup = (uint64_t **)calloc((size_t)n, sizeof(uint64_t *));
  if (!c->dom || !c->deg || !c->nbr || !c->sup) { orc_wfree(c); return NULL; }
  for (int x = 0; x < n; ++x) c->dom[x] = dom[x];
  return c;
}

static int walloc_arcs(orc_wcsp *c) {
  for (int x = 0; x < c->n; ++x) {
    size_t k = (size_t)(c->deg[x] > 0 ? c->deg[x] : 1);
    c->nbr[x] = (int *)malloc(k * sizeof(int));
    c->sup[x] = (uint64_t *)calloc(k * (size_t)c->dom[x] * (size_t)c->wq, sizeof(uint64_t));
    if (!c->nbr[x] || !c->sup[x]) return -1;
  }
  return 0;
}

static int warc_index(const orc_wcsp *c, int x, int y) {
  for (int k = 0; k < c->deg[x]; ++k) if (c->nbr[x][k] == y) return k;
  return -1;
}

int orc_wq(const orc_wcsp *c) { return c->wq; }

/*
 * Explicit relations: constraint r on (xs[r], ys[r]); row a of rel(c_{xs,ys})
 * is the wq-word bitset rows[(r*row_stride + a)*wq .. +wq) (bit b set iff
 * (a,b) allowed), wq = ceil(max dom / 64).  Domain sizes 1..256.
 */
orc_wcsp *orc_wbuild(int n, const int *dom, int n_rel, const int *xs, const int *ys,
                     const uint64_t *rows, int row_stride) {
  if (n < 1) return NULL;
  for (int x = 0; x < n; ++x)
    if (dom[x] < 1 || dom[x] > 256) return NULL;
  orc_wcsp *c = walloc(n, dom);
  if (!c) return NULL;
  const int wq = c->wq;
  for (int r = 0; r < n_rel; ++r) {
    int x = xs[r], y = ys[r];
    if (x < 0 || y < 0 || x >= n || y >= n || x == y) { orc_wfree(c); return NULL; }
    c->deg[x]++; c->deg[y]++;
  }
  if (walloc_arcs(c)) { orc_wfree(c); return NULL; }
  int *fill = (int *)calloc((size_t)n, sizeof(int));
  for (int r = 0; r < n_rel; ++r) {
    c->nbr[xs[r]][fill[xs[r]]++] = ys[r];
    c->nbr[ys[r]][fill[ys[r]]++] = xs[r];
  }
  free(fill);
  for (int x = 0; x < n; ++x) {
    qsort(c->nbr[x], (size_t)c->deg[x], sizeof(int), cmp_int);
    for (int k = 1; k < c->deg[x]; ++k)
      if (c->nbr[x][k] == c->nbr[x][k - 1]) { orc_wfree(c); return NULL; }
  }
  for (int r = 0; r < n_rel; ++r) {
    int x = xs[r], y = ys[r];
    int kx = warc_index(c, x, y), ky = warc_index(c, y, x);
    for (int a = 0; a < row_stride; ++a) {
      const uint64_t *row = rows + ((size_t)r * (size_t)row_stride + (size_t)a) * (size_t)wq;
      for (int b = 0; b < 64 * wq; ++b) {
        if (!wbit(row, b)) continue;
        if (a >= dom[x] || b >= dom[y]) { orc_wfree(c); return NULL; } /* bits beyond the domains */
        /* arc x -> y: c_xy|(x,a) = row a; arc y -> x: the transpose */
        wset(c->sup[x] + ((size_t)kx * dom[x] + a) * wq, b);
        wset(c->sup[y] + ((size_t)ky * dom[y] + b) * wq, a);
      }
    }
  }
  return c;
}

/*
 * The seeded random instance of synth/csp_synth.h, uniform domain d <= 256,
 * with arcs only for the variables x in [x_lo, x_hi) (all their neighbours y);
 * the full instance is x_lo = 0, x_hi = n.  A partial build serves sampled CPU
 * timing at sizes the full instance does not fit (orc_wpass_block only).
 */
orc_wcsp *orc_wbuild_synth_block(int n, int d, uint64_t dens_q32, uint32_t t_q16, uint64_t seed, int x_lo, int x_hi) {
  if (n < 1 || d < 1 || d > 256 || x_lo < 0 || x_hi > n || x_lo > x_hi) return NULL;
  int *dom = (int *)malloc((size_t)n * sizeof(int));
  for (int x = 0; x < n; ++x) dom[x] = d;
  orc_wcsp *c = walloc(n, dom);
  free(dom);
  if (!c) return NULL;
  const int wq = c->wq;
  for (int x = x_lo; x < x_hi; ++x)
    for (int y = 0; y < n; ++y) {
      if (y == x) continue;
      int lo = x < y ? x : y, hi = x < y ? y : x;
      if (synth_present(seed, (uint32_t)n, (uint32_t)lo, (uint32_t)hi, dens_q32)) c->deg[x]++;
    }
  if (walloc_arcs(c)) { orc_wfree(c); return NULL; }
  for (int x = x_lo; x < x_hi; ++x) {
    int k = 0;
    for (int y = 0; y < n; ++y) {
      if (y == x) continue;
      int lo = x < y ? x : y, hi = x < y ? y : x;
      if (synth_present(seed, (uint32_t)n, (uint32_t)lo, (uint32_t)hi, dens_q32)) c->nbr[x][k++] = y;
    }
  }
  for (int x = x_lo; x < x_hi; ++x)
    for (int k = 0; k < c->deg[x]; ++k) {
      int y = c->nbr[x][k];
      for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) {
          /* (a,b) in c_xy: for x < y the generator's cell; for x > y the transpose of c_yx */
          int ok = x < y ? synth_allowed(seed, (uint32_t)n, (uint32_t)d, (uint32_t)x, (uint32_t)y, (uint32_t)a,
                                         (uint32_t)b, t_q16)
                         : synth_allowed(seed, (uint32_t)n, (uint32_t)d, (uint32_t)y, (uint32_t)x, (uint32_t)b,
                                         (uint32_t)a, t_q16);
          if (ok) wset(c->sup[x] + ((size_t)k * d + a) * wq, b);
        }
    }
  return c;
}

orc_wcsp *orc_wbuild_synth(int n, int d, uint64_t dens_q32, uint32_t t_q16, uint64_t seed) {
  return orc_wbuild_synth_block(n, d, dens_q32, t_q16, seed, 0, n);
}

/* c_xy|(x,a) ∩ D(y) ≠ ∅ over wq words. */
static int wmeets(const uint64_t *s, const uint64_t *Dy, int wq) {
  for (int w = 0; w < wq; ++w) if (s[w] & Dy[w]) return 1;
  return 0;
}

static int wempty(const uint64_t *v, int wq) {
  for (int w = 0; w < wq; ++w) if (v[w]) return 0;
  return 1;
}

/* O1w: orc_rac with wq-word domains (same loop, same readings R1-R7). */
int orc_rac_wide(const orc_wcsp *c, const uint64_t *d_in, uint64_t *d_out, int *iterations,
                 int32_t *removed_at, int full) {
  const int n = c->n, wq = c->wq;
  const size_t nw = (size_t)n * wq;
  uint64_t *prev = (uint64_t *)calloc(nw, sizeof(uint64_t));
  uint64_t *next = (uint64_t *)calloc(nw, sizeof(uint64_t));
  memcpy(prev, d_in, nw * sizeof(uint64_t));
  if (removed_at) memset(removed_at, 0, (size_t)n * 64 * wq * sizeof(int32_t));
  int k = 0, status = ORC_OK;
  for (;;) {
    ++k;
    memcpy(next, prev, nw * sizeof(uint64_t));
    for (int x = 0; x < n; ++x)
      for (int a = 0; a < c->dom[x]; ++a) {
        if (!wbit(prev + (size_t)x * wq, a)) continue;
        for (int kk = 0; kk < c->deg[x]; ++kk) {
          int y = c->nbr[x][kk];
          const uint64_t *s = c->sup[x] + ((size_t)kk * c->dom[x] + a) * wq; /* c_xy|(x,a) */
          if (!wmeets(s, prev + (size_t)y * wq, wq)) {                         /* ∩ D_{k-1}(y) = ∅ */
            next[(size_t)x * wq + (a >> 6)] &= ~(1ULL << (a & 63));
            if (removed_at) removed_at[(size_t)x * 64 * wq + a] = k;
            break;
          }
        }
      }
    int wipe = 0, changed = 0;
    for (int x = 0; x < n; ++x) {
      if (wempty(next + (size_t)x * wq, wq)) wipe = 1;
      for (int w = 0; w < wq; ++w) if (next[(size_t)x * wq + w] != prev[(size_t)x * wq + w]) changed = 1;
    }
    memcpy(prev, next, nw * sizeof(uint64_t));
    if (wipe && !full) { status = ORC_WIPEOUT; break; } /* Alg. 1 */
    if (!changed) { status = wipe ? ORC_WIPEOUT : ORC_OK; break; }
  }
  memcpy(d_out, prev, nw * sizeof(uint64_t));
  *iterations = k;
  free(prev); free(next);
  return status;
}

/*
 * O6w: Alg. 2 backtracking search on wide domains,
 * the same recursion as orc_search over O1w (engine "full": by Prop. 2 the
 * seeded call tensorAC(Vars, [idx]) of line 392 follows the same trajectory
 * after an assignment on an arc-consistent state, reading R12): min-domain
 * variable (lowest index on ties), ascending values, assignment on a copy of
 * the parent's domains.  stats as orc_search; returns 0 solution, 1 unsat,
 * 2 budget exhausted.
 */
typedef struct {
  const orc_wcsp *c;
  int64_t budget;
  int all, full;
  int64_t *stats;
  int32_t *solution;
  char *assigned;
  int found, out_of_budget;
} orc_wsearch_ctx;

static int wcount(const uint64_t *v, int wq) {
  int k = 0;
  for (int w = 0; w < wq; ++w) k += popc64(v[w]);
  return k;
}

static int orc_wdfs(orc_wsearch_ctx *s, const uint64_t *D, int level) {
  const orc_wcsp *c = s->c;
  const int n = c->n, wq = c->wq;
  const size_t nw = (size_t)n * wq;
  int idx = -1, best = 1 << 30;
  for (int x = 0; x < n; ++x) {
    if (s->assigned[x]) continue;
    const int k = wcount(D + (size_t)x * wq, wq);
    if (k < best) { best = k; idx = x; }
  }
  s->assigned[idx] = 1;
  uint64_t *child = (uint64_t *)malloc(nw * sizeof(uint64_t));
  uint64_t *out = (uint64_t *)malloc(nw * sizeof(uint64_t));
  int stop = 0;
  for (int v = 0; v < 64 * wq && !stop; ++v) {
    if (!wbit(D + (size_t)idx * wq, v)) continue;
    if (s->budget > 0 && s->stats[0] >= s->budget) { s->out_of_budget = 1; stop = 1; break; }
    memcpy(child, D, nw * sizeof(uint64_t));
    for (int w = 0; w < wq; ++w) child[(size_t)idx * wq + w] = 0;
    wset(child + (size_t)idx * wq, v); /* assign, lines 410-416 */
    int it = 0;
    const int st = orc_rac_wide(c, child, out, &it, NULL, s->full);
    s->stats[0]++;
    s->stats[1] += it;
    if (st == ORC_WIPEOUT) { s->stats[2]++; continue; }
    if (level + 1 > s->stats[4]) s->stats[4] = level + 1;
    if (level + 1 == n) {
      s->stats[3]++;
      if (!s->found && s->solution)
        for (int x = 0; x < n; ++x)
          for (int b = 0; b < 64 * wq; ++b)
            if (wbit(out + (size_t)x * wq, b)) { s->solution[x] = b; break; }
      s->found = 1;
      if (!s->all) stop = 1;
      continue;
    }
    if (orc_wdfs(s, out, level + 1)) stop = 1;
  }
  free(child); free(out);
  s->assigned[idx] = 0;
  return stop;
}

int orc_wsearch(const orc_wcsp *c, const uint64_t *d_in, int64_t max_assignments, int all, int full,
                int32_t *solution, int64_t *stats) {
  const int n = c->n;
  for (int k = 0; k < 6; ++k) stats[k] = 0;
  uint64_t *root = (uint64_t *)malloc((size_t)n * c->wq * sizeof(uint64_t));
  int it = 0;
  const int st = orc_rac_wide(c, d_in, root, &it, NULL, full);
  stats[5] = it;
  if (st == ORC_WIPEOUT) { free(root); return 1; }
  orc_wsearch_ctx s = {c, max_assignments, all, full, stats, solution, NULL, 0, 0};
  s.assigned = (char *)calloc((size_t)n, 1);
  orc_wdfs(&s, root, 0);
  free(s.assigned);
  free(root);
  if (s.out_of_budget) return 2;
  return s.found ? 0 : 1;
}

/* Arc consistency by definition on wide domains: 1 iff AC and no empty domain. */
int orc_wis_ac(const orc_wcsp *c, const uint64_t *D) {
  const int wq = c->wq;
  for (int x = 0; x < c->n; ++x) {
    if (wempty(D + (size_t)x * wq, wq)) return 0;
    for (int a = 0; a < c->dom[x]; ++a) {
      if (!wbit(D + (size_t)x * wq, a)) continue;
      for (int k = 0; k < c->deg[x]; ++k)
        if (!wmeets(c->sup[x] + ((size_t)k * c->dom[x] + a) * wq, D + (size_t)c->nbr[x][k] * wq, wq)) return 0;
    }
  }
  return 1;
}

/*
 * Textbook AC-3 on wide domains: a FIFO of arcs (x, y); revising
 * removes from D(x) every a with c_xy|(x,a) ∩ D(y) = ∅; a change re-queues
 * every arc (z, x), z ≠ y.  Runs to the fixpoint (FULL semantics).
 * Returns ORC_WIPEOUT if some domain ends empty.
 */
int orc_wac3(const orc_wcsp *c, const uint64_t *d_in, uint64_t *d_out) {
  const int n = c->n, wq = c->wq;
  memcpy(d_out, d_in, (size_t)n * wq * sizeof(uint64_t));
  size_t narcs = 0;
  for (int x = 0; x < n; ++x) narcs += (size_t)c->deg[x];
  size_t cap = narcs + 1, head = 0, count = 0;
  int *qx = (int *)malloc(cap * sizeof(int)), *qk = (int *)malloc(cap * sizeof(int));
  char *inq = (char *)calloc(cap, 1);
  size_t *base = (size_t *)calloc((size_t)n + 1, sizeof(size_t));
  for (int x = 0; x < n; ++x) base[x + 1] = base[x] + (size_t)c->deg[x];
  for (int x = 0; x < n; ++x)
    for (int k = 0; k < c->deg[x]; ++k) {
      qx[(head + count) % cap] = x; qk[(head + count) % cap] = k; ++count;
      inq[base[x] + k] = 1;
    }
  while (count) {
    int x = qx[head], k = qk[head];
    head = (head + 1) % cap; --count;
    inq[base[x] + k] = 0;
    int y = c->nbr[x][k], changed = 0;
    for (int a = 0; a < c->dom[x]; ++a) {
      if (!wbit(d_out + (size_t)x * wq, a)) continue;
      if (!wmeets(c->sup[x] + ((size_t)k * c->dom[x] + a) * wq, d_out + (size_t)y * wq, wq)) {
        d_out[(size_t)x * wq + (a >> 6)] &= ~(1ULL << (a & 63));
        changed = 1;
      }
    }
    if (!changed) continue;
    for (int j = 0; j < c->deg[x]; ++j) {
      int z = c->nbr[x][j];
      if (z == y) continue;
      int kz = warc_index(c, z, x);
      if (!inq[base[z] + kz]) {
        qx[(head + count) % cap] = z; qk[(head + count) % cap] = kz; ++count;
        inq[base[z] + kz] = 1;
      }
    }
  }
  free(qx); free(qk); free(inq); free(base);
  for (int x = 0; x < n; ++x)
    if (wempty(d_out + (size_t)x * wq, wq)) return ORC_WIPEOUT;
  return ORC_OK;
}

/* One Eq. 1 step over the rows of x in [x_lo, x_hi) against D:
 * out[x*wq + w] = D(x) minus the values with an empty support on some c_xy.
 * Returns the number of values removed. */
int64_t orc_wpass_block(const orc_wcsp *c, const uint64_t *D, int x_lo, int x_hi, uint64_t *out) {
  const int wq = c->wq;
  int64_t removed = 0;
  for (int x = x_lo; x < x_hi; ++x) {
    for (int w = 0; w < wq; ++w) out[(size_t)x * wq + w] = D[(size_t)x * wq + w];
    for (int a = 0; a < c->dom[x]; ++a) {
      if (!wbit(D + (size_t)x * wq, a)) continue;
      for (int k = 0; k < c->deg[x]; ++k)
        if (!wmeets(c->sup[x] + ((size_t)k * c->dom[x] + a) * wq, D + (size_t)c->nbr[x][k] * wq, wq)) {
          out[(size_t)x * wq + (a >> 6)] &= ~(1ULL << (a & 63));
          ++removed;
          break;
        }
    }
  }
  return removed;
}

/* ======================================================================== */
/*
 * O7: exact-trajectory certificate.  Given D_in, the
 * claimed output D_out, the claimed removal epochs eps(x,a) (0 = kept), the
 * claimed iteration count K and status, accept iff they are exactly what the
 * RAC recurrence (Eq. 1, with Alg. 1's loop control,
 * lines 198-210, readings R1-R7) produces -- without running the recurrence.
 *
 * The epochs define the claimed trajectory
 *     D_s = { (y,b) in D_in : eps(y,b) = 0 or eps(y,b) > s },   s = 0..K
 * (D_0 = D_in).  Eq. 1 removes (x,a) at pass t iff (x,a) in D_{t-1} and some
 * declared c_xy in C_x has c_xy|(x,a) ∩ D_{t-1}(y) = ∅ (R1, R2).  So the claim is
 * the recurrence's iff, for every (x,a) in D_in:
 *   removed at e >= 1:  (L1) some declared c_xy has c_xy|(x,a) ∩ D_{e-1}(y) = ∅
 *                            -- the Eq. 1 removal test at pass e; this is
 *                            Lemma 1 (lines 79-82): all supports were removed
 *                            before e;
 *                       (P2) if e >= 2, every declared c_xy has
 *                            c_xy|(x,a) ∩ D_{e-2}(y) ≠ ∅ -- (x,a) survived pass
 *                            e-1, so it is removed exactly at e (Prop. 2, lines
 *                            130-143: removals at step e are caused by removals
 *                            at step e-1);
 *   kept:               (AC) every declared c_xy has c_xy|(x,a) ∩ D_{K-1}(y) ≠ ∅
 *                            (it survives the last pass; D is monotone, so
 *                            every earlier pass too);
 * and the loop control matches Alg. 1 (R3, R5):
 *   every pass t < K removed something (otherwise the loop ends at t);
 *   status OK:        D_K has no empty domain and pass K removed nothing
 *                     (Prop. 1 end condition, line 125: D_K is arc consistent);
 *   status WIPEOUT, stop mode: D_K has an empty domain and D_{K-1} has none
 *                     unless K = 1 (an empty domain in D_in: one pass, R7);
 *   status WIPEOUT, full mode: pass K removed nothing and D_K has an empty domain.
 * Also D_out = D_K, epochs lie in [1, K] exactly on D_in \ D_out, D_out ⊆ D_in.
 * By induction on t the set {eps = t} is determined by {eps < t}, so exactly
 * one claim passes: the recurrence's own trajectory.
 *
 * Layout of the checks: for each y the level bitsets E[y][s] = D_s(y) (wq words
 * each).  Domain states are wq words per variable (wq = 1: the one-word layout);
 * epochs removed_at[x*64*wq + a].
 *
 * Return codes: 0 accepted; 2 D_out ⊄ D_in or bits beyond dom; 3 epochs
 * inconsistent with D_in / D_out / K; 5 (L1) fails: a removal without an empty
 * support set at its pass; 6 (P2) fails: the value should have gone one pass
 * earlier; 7 (AC) fails: a kept value without support in D_{K-1}; 8 loop
 * control (K, status) inconsistent; -1 bad arguments / out of memory.
 */
static int cert_word_bit(const uint64_t *v, int b) { return (int)((v[b >> 6] >> (b & 63)) & 1ULL); }

/* Global part: epochs against D_in / D_out / K, the level bitsets E, and the
 * loop-control rules.  E = [n][K+1][wq], allocated here. */
static int cert_global(int n, const int *dom, int wq, const uint64_t *d_in, const uint64_t *d_out,
                       const int32_t *eps, int K, int status, int full, uint64_t **E_out) {
  *E_out = NULL;
  if (K < 0 || (status != ORC_OK && status != ORC_WIPEOUT)) return 8;
  const size_t nw = (size_t)n * wq;
  for (size_t i = 0; i < nw; ++i)
    if (d_out[i] & ~d_in[i]) return 2;
  for (int x = 0; x < n; ++x)
    for (int b = 0; b < 64 * wq; ++b) {
      const int in = cert_word_bit(d_in + (size_t)x * wq, b), out = cert_word_bit(d_out + (size_t)x * wq, b);
      const int32_t e = eps[(size_t)x * 64 * wq + b];
      if (b >= dom[x] && (in || e != 0)) return 2;
      if (in && !out) { if (e < 1 || e > K) return 3; }
      else if (e != 0) return 3;
    }
  if (K == 0) return 8; /* every enforcement runs at least one pass (R3) */
  uint64_t *E = (uint64_t *)calloc((size_t)n * (size_t)(K + 1) * wq, sizeof(uint64_t));
  if (!E) return -1;
  int *removed_at_t = (int *)calloc((size_t)K + 2, sizeof(int)); /* number of values with eps = t */
  int *empty_at_s = (int *)calloc((size_t)K + 1, sizeof(int));   /* D_s has an empty domain */
  if (!removed_at_t || !empty_at_s) { free(E); free(removed_at_t); free(empty_at_s); return -1; }
  for (int y = 0; y < n; ++y)
    for (int b = 0; b < dom[y]; ++b) {
      if (!cert_word_bit(d_in + (size_t)y * wq, b)) continue;
      const int32_t e = eps[(size_t)y * 64 * wq + b];
      if (e > 0) removed_at_t[e]++;
      for (int s = 0; s <= K; ++s)
        if (e == 0 || e > s) E[((size_t)y * (K + 1) + s) * wq + (b >> 6)] |= 1ULL << (b & 63);
    }
  for (int s = 0; s <= K; ++s)
    for (int y = 0; y < n; ++y) {
      int any = 0;
      for (int w = 0; w < wq; ++w) any |= E[((size_t)y * (K + 1) + s) * wq + w] != 0;
      if (!any) { empty_at_s[s] = 1; break; }
    }
  int bad = 0;
  for (int t = 1; t < K; ++t)
    if (removed_at_t[t] == 0) bad = 1; /* the loop would have ended at t */
  if (status == ORC_OK) {
    if (empty_at_s[K] || removed_at_t[K] != 0) bad = 1;
  } else if (!full) {
    if (!empty_at_s[K] || (K > 1 && empty_at_s[K - 1])) bad = 1;
  } else {
    if (!empty_at_s[K] || removed_at_t[K] != 0) bad = 1;
  }
  free(removed_at_t);
  free(empty_at_s);
  if (bad) { free(E); return 8; }
  *E_out = E;
  return 0;
}

/* c_xy|(x,a) ∩ D_s(y) ≠ ∅ for the wq-word support set `sup`. */
static int cert_meets(const uint64_t *sup, const uint64_t *E, int y, int K, int s, int wq) {
  const uint64_t *Ds = E + ((size_t)y * (K + 1) + s) * wq;
  for (int w = 0; w < wq; ++w)
    if (sup[w] & Ds[w]) return 1;
  return 0;
}

/* Per-variable part: every (x,a) in D_in against the (L1), (P2), (AC) rules.
 * nbr[k] (k < deg) are the constrained neighbours of x, sup[((size_t)k*dom_x +
 * a)*wq + w] the support sets c_{x,nbr[k]}|(x,a). */
static int cert_var(int x, int dom_x, int deg, const int *nbr, const uint64_t *sup, int wq, const uint64_t *E,
                    const uint64_t *d_in, const int32_t *eps, int K) {
  for (int a = 0; a < dom_x; ++a) {
    if (!cert_word_bit(d_in + (size_t)x * wq, a)) continue;
    const int32_t e = eps[(size_t)x * 64 * wq + a];
    if (e == 0) { /* kept: supported in D_{K-1} on every declared constraint */
      for (int k = 0; k < deg; ++k)
        if (!cert_meets(sup + ((size_t)k * dom_x + a) * wq, E, nbr[k], K, K - 1, wq)) return 7;
    } else {
      int l1 = 0;
      for (int k = 0; k < deg; ++k) {
        const uint64_t *s = sup + ((size_t)k * dom_x + a) * wq;
        if (!cert_meets(s, E, nbr[k], K, e - 1, wq)) l1 = 1;                 /* (L1) */
        if (e >= 2 && !cert_meets(s, E, nbr[k], K, e - 2, wq)) return 6;      /* (P2) */
      }
      if (!l1) return 5;
    }
  }
  return 0;
}

int orc_certify_trajectory(const orc_csp *c, const uint64_t *d_in, const uint64_t *d_out, const int32_t *removed_at,
                           int iterations, int status, int full) {
  uint64_t *E = NULL;
  int rc = cert_global(c->n, c->dom, 1, d_in, d_out, removed_at, iterations, status, full, &E);
  if (rc) return rc;
  for (int x = 0; x < c->n && rc == 0; ++x)
    rc = cert_var(x, c->dom[x], c->deg[x], c->nbr[x], c->sup[x], 1, E, d_in, removed_at, iterations);
  free(E);
  return rc;
}

int orc_wcertify_trajectory(const orc_wcsp *c, const uint64_t *d_in, const uint64_t *d_out,
                            const int32_t *removed_at, int iterations, int status, int full) {
  uint64_t *E = NULL;
  int rc = cert_global(c->n, c->dom, c->wq, d_in, d_out, removed_at, iterations, status, full, &E);
  if (rc) return rc;
  for (int x = 0; x < c->n && rc == 0; ++x)
    rc = cert_var(x, c->dom[x], c->deg[x], c->nbr[x], c->sup[x], c->wq, E, d_in, removed_at, iterations);
  free(E);
  return rc;
}

/*
 * The same certificate for the seeded random instance of synth/csp_synth.h
 * (uniform d <= 256) at sizes where the oracle's instance does not fit in host
 * memory (C4: 32.8 GB of support sets).  Each constrained pair {x < y} is
 * regenerated once from the generator as its d x d cell matrix; its rows are the
 * support sets c_xy|(x,a) and its columns the c_yx|(y,b).  The per-value rules
 * are OR-reductions over the constraints, so every pair contributes flags
 *   F_L1 : this constraint has c|(x,a) ∩ D_{e-1}(y) = ∅         (wanted for e >= 1)
 *   F_P2 : this constraint has c|(x,a) ∩ D_{e-2}(y) = ∅         (forbidden for e >= 2)
 *   F_AC : this constraint has c|(x,a) ∩ D_{K-1}(y) = ∅         (forbidden for kept)
 * to both endpoints; the rules are checked once all pairs are in (the same
 * rules as cert_var).  Pairs are spread over `threads` OpenMP threads (0 = all)
 * with per-thread flag arrays OR-ed together, so the verdict does not depend on
 * the thread count.
 */
#define CERT_F_L1 1
#define CERT_F_P2 2
#define CERT_F_AC 4

static void cert_pair_side(const uint64_t *rowsup /* [d][wq] supports of the side's values */, int x, int y, int d,
                           int wq, const uint64_t *E, const uint64_t *d_in, const int32_t *eps, int K,
                           uint8_t *flags /* [n][64*wq] */) {
  for (int a = 0; a < d; ++a) {
    if (!cert_word_bit(d_in + (size_t)x * wq, a)) continue;
    const int32_t e = eps[(size_t)x * 64 * wq + a];
    const uint64_t *sp = rowsup + (size_t)a * wq;
    uint8_t f = 0;
    if (e == 0) {
      if (!cert_meets(sp, E, y, K, K - 1, wq)) f |= CERT_F_AC;
    } else {
      if (!cert_meets(sp, E, y, K, e - 1, wq)) f |= CERT_F_L1;
      if (e >= 2 && !cert_meets(sp, E, y, K, e - 2, wq)) f |= CERT_F_P2;
    }
    flags[(size_t)x * 64 * wq + a] |= f;
  }
}

int orc_certify_trajectory_synth(int n, int d, uint64_t dens_q32, uint32_t t_q16, uint64_t seed,
                                 const uint64_t *d_in, const uint64_t *d_out, const int32_t *removed_at,
                                 int iterations, int status, int full, int threads) {
  if (n < 1 || d < 1 || d > 256) return -1;
  const int wq = (d + 63) / 64, K = iterations;
  int *dom = (int *)malloc((size_t)n * sizeof(int));
  if (!dom) return -1;
  for (int x = 0; x < n; ++x) dom[x] = d;
  uint64_t *E = NULL;
  int rc = cert_global(n, dom, wq, d_in, d_out, removed_at, iterations, status, full, &E);
  free(dom);
  if (rc) return rc;
  const size_t nv = (size_t)n * 64 * wq;
  uint8_t *flags = (uint8_t *)calloc(nv, 1);
  if (!flags) { free(E); return -1; }
  const int q = (d + 3) / 4;
  int oom = 0;
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel
#endif
  {
    uint8_t *fl = (uint8_t *)calloc(nv, 1);               /* this thread's flags */
    uint64_t *fw = (uint64_t *)malloc((size_t)d * wq * 8); /* fw[a] = c_xy|(x,a) (rows)    */
    uint64_t *bw = (uint64_t *)malloc((size_t)d * wq * 8); /* bw[b] = c_yx|(y,b) (columns) */
    const int ok = fl && fw && bw;
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 4)
#endif
    for (int x = 0; x < n; ++x) {
      if (!ok) continue;
      for (int y = x + 1; y < n; ++y) {
        if (!synth_present(seed, (uint32_t)n, (uint32_t)x, (uint32_t)y, dens_q32)) continue;
        memset(fw, 0, (size_t)d * wq * 8);
        memset(bw, 0, (size_t)d * wq * 8);
        const uint64_t pk = synth_pair_key(seed, (uint32_t)n, (uint32_t)x, (uint32_t)y);
        for (int a = 0; a < d; ++a)
          for (int bq = 0; bq < q; ++bq) {
            const uint64_t h = synth_cell_word_pk(pk, (uint32_t)d, (uint32_t)a, (uint32_t)bq);
            for (int j = 0; j < 4 && 4 * bq + j < d; ++j) {
              const int b = 4 * bq + j;
              const uint64_t allowed = ((h >> (16 * j)) & 0xFFFFULL) >= t_q16; /* (a,b) in rel(c_xy) */
              fw[(size_t)a * wq + (b >> 6)] |= allowed << (b & 63);
              bw[(size_t)b * wq + (a >> 6)] |= allowed << (a & 63);
            }
          }
        cert_pair_side(fw, x, y, d, wq, E, d_in, removed_at, K, fl);
        cert_pair_side(bw, y, x, d, wq, E, d_in, removed_at, K, fl);
      }
    }
#ifdef _OPENMP
#pragma omp critical
#endif
    {
      if (!ok) oom = 1;
      else
        for (size_t i = 0; i < nv; ++i) flags[i] |= fl[i];
    }
    free(fl);
    free(fw);
    free(bw);
  }
  free(E);
  if (oom) { free(flags); return -1; }
  /* the per-value rules of cert_var, in the same order of precedence */
  int err = 0;
  for (int x = 0; x < n && !err; ++x)
    for (int a = 0; a < d && !err; ++a) {
      if (!cert_word_bit(d_in + (size_t)x * wq, a)) continue;
      const int32_t e = removed_at[(size_t)x * 64 * wq + a];
      const uint8_t f = flags[(size_t)x * 64 * wq + a];
      if (e == 0) { if (f & CERT_F_AC) err = 7; }
      else if (f & CERT_F_P2) err = 6;
      else if (!(f & CERT_F_L1)) err = 5;
    }
  free(flags);
  return err;
}
