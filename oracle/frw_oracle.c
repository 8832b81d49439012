/*
 * frw_oracle.c -- CPU restatement of the reference FRW/MicroWalk hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see frw_oracle.h).  Plain C99 + pthreads,
 * compiled with -O2 -ffp-contract=off.  Each block cites the reference
 * file:line (relative to /root/reference/proj) it restates.  Exceptions of
 * the reference become negative status codes plus frwo_last_error().
 *
 * Deliberate differences from the reference (documented in DESIGN.md):
 *  - the SGF solve is a matrix-free Jacobi-PCG on s_ii (same algorithm as
 *    Eigen::ConjugateGradient with DiagonalPreconditioner, sgf.cpp:162-211)
 *    without the SimplicialLDLT fallback; results agree with the reference
 *    to ~1e-10 relative, not bit for bit (Eigen vectorises its dot products).
 *  - masked (conductor) grids are supported by MicroWalk but not by the
 *    solver (the cached SGFs of the hot path are never masked).
 */
#define _GNU_SOURCE
#include "frw_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static __thread char g_err[512];
static void set_err(const char *msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
}
const char *frwo_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------ */
/* rng.hpp:12-40  SplitMix64                                                */

#define GAMMA 0x9E3779B97F4A7C15ULL

uint64_t frwo_mix(uint64_t z) {
  z += GAMMA;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
/* rng.hpp:16-17: state = mix(mix(seed) + (stream+1)*gamma) */
uint64_t frwo_stream_state(uint64_t seed, uint64_t stream) {
  return frwo_mix(frwo_mix(seed) + (stream + 1) * GAMMA);
}
uint64_t frwo_next(uint64_t *s) {
  *s += GAMMA;
  return frwo_mix(*s);
}
/* rng.hpp:25 */
double frwo_uniform(uint64_t *s) {
  return (double)(frwo_next(s) >> 11) * 0x1.0p-53;
}

/* ------------------------------------------------------------------------ */
/* sgf.hpp:24-61, sgf.cpp:13-55  lattice and panel conventions              */

static const int kDirAxis[6] = {0, 0, 1, 1, 2, 2};
static const int kDirSign[6] = {-1, +1, -1, +1, -1, +1};

int frwo_surface_panel_of(int n, int i, int j, int k, int dir) {
  int u, v;
  switch (kDirAxis[dir]) {
    case 0: u = j; v = k; break;
    case 1: u = i; v = k; break;
    default: u = i; v = j; break;
  }
  return (dir * n + v) * n + u; /* sgf.hpp:34-36 */
}

void frwo_surface_panel_center(const double c[3], double h, int n, int panel,
                               double p[3]) {
  const int face = panel / (n * n);
  const int rem = panel % (n * n);
  const int u = rem % n, v = rem / n;
  const int axis = kDirAxis[face];
  const double pitch = 2.0 * h / n;
  p[axis] = c[axis] + kDirSign[face] * h;
  const int b1 = axis == 0 ? 1 : 0;
  const int b2 = axis == 2 ? 1 : 2;
  p[b1] = c[b1] - h + (u + 0.5) * pitch;
  p[b2] = c[b2] - h + (v + 0.5) * pitch;
}

/* microwalk.hpp:39-44 */
void frwo_transit_cube(const double p[3], double hw, int n, double oc[3],
                       double *oh) {
  if (n % 2 == 1) {
    oc[0] = p[0]; oc[1] = p[1]; oc[2] = p[2];
    *oh = hw;
    return;
  }
  const double delta = hw / (n + 1);
  const double h = (hw - delta) * (1.0 - 1e-12);
  oc[0] = p[0] + delta; oc[1] = p[1] + delta; oc[2] = p[2] + delta;
  *oh = h;
}

/* microwalk.cpp:25-30 and geometry.hpp:166-171 (same expression) */
static inline void voxel_center(const double c[3], double h, int n, int i,
                                int j, int k, double out[3]) {
  const double p = 2.0 * h / n;
  out[0] = c[0] - h + (i + 0.5) * p;
  out[1] = c[1] - h + (j + 0.5) * p;
  out[2] = c[2] - h + (k + 0.5) * p;
}

/* ------------------------------------------------------------------------ */
/* geometry.cpp:31-80  box queries                                          */

static inline double dmax(double a, double b) { return a < b ? b : a; }
static inline double dmin(double a, double b) { return b < a ? b : a; }

static inline int box_contains(const double *b, const double p[3]) {
  return p[0] >= b[0] && p[0] <= b[3] && p[1] >= b[1] && p[1] <= b[4] &&
         p[2] >= b[2] && p[2] <= b[5];
}
static inline double box_cheb_to(const double *b, const double p[3]) {
  double d = 0;
  for (int a = 0; a < 3; ++a) d = dmax(d, dmax(b[a] - p[a], p[a] - b[3 + a]));
  return dmax(d, 0.0);
}
static inline double box_cheb_to_wall(const double *b, const double p[3]) {
  double d = INFINITY;
  for (int a = 0; a < 3; ++a) d = dmin(d, dmin(p[a] - b[a], b[3 + a] - p[a]));
  return d;
}

int frwo_permittivity_at(const frwo_structure *s, const double p[3],
                         double *eps) {
  if (!box_contains(s->world, p)) {
    set_err("permittivity_at: point outside world box");
    return -1;
  }
  double e = s->background_eps;
  for (int d = 0; d < s->n_diel; ++d)
    if (box_contains(s->diel_box + 6 * d, p)) e = s->diel_eps[d];
  *eps = e;
  return 0;
}

int frwo_conductor_at(const frwo_structure *s, const double p[3], double tol) {
  for (int c = 0; c < s->n_cond; ++c)
    if (box_cheb_to(s->cond_box + 6 * c, p) <= tol) return c;
  return -1;
}

int frwo_max_free_cube(const frwo_structure *s, const double p[3], double *hw,
                       int *nearest) {
  double h = box_cheb_to_wall(s->world, p);
  int near = -1;
  if (h <= 0) {
    set_err("max_free_cube: point not inside the world");
    return -1;
  }
  for (int c = 0; c < s->n_cond; ++c) {
    const double d = box_cheb_to(s->cond_box + 6 * c, p);
    if (d <= 0) {
      set_err("max_free_cube: point inside conductor");
      return -1;
    }
    if (d <= h) { /* ties go to the conductor */
      h = d;
      near = c;
    }
  }
  *hw = h;
  if (nearest) *nearest = near;
  return 0;
}

/* geometry.cpp:15-19 */
static inline int eps_equal(double a, double b) {
  return fabs(a - b) <= 1e-9 * dmax(fabs(a), fabs(b));
}

/* geometry.cpp:357-396 */
int frwo_stratified_profile(const frwo_structure *s, const double c[3],
                            double h, int n, double *layers) {
  double cb[6] = {c[0] - h, c[1] - h, c[2] - h, c[0] + h, c[1] + h, c[2] + h};
  int nhits = 0;
  int stack_hits[64];
  int *hits = s->n_diel <= 64 ? stack_hits : malloc(sizeof(int) * s->n_diel);
  for (int d = 0; d < s->n_diel; ++d) {
    const double *b = s->diel_box + 6 * d;
    /* geometry.hpp:49-52 intersects_open */
    if (b[0] < cb[3] && cb[0] < b[3] && b[1] < cb[4] && cb[1] < b[4] &&
        b[2] < cb[5] && cb[2] < b[5])
      hits[nhits++] = d;
  }
  int axis = -1;
  if (nhits == 0) {
    axis = 0;
  } else {
    for (int a = 0; a < 3 && axis < 0; ++a) {
      int covers = 1;
      for (int q = 0; q < nhits && covers; ++q) {
        const double *b = s->diel_box + 6 * hits[q];
        for (int pp = 1; pp <= 2 && covers; ++pp) {
          const int bb = (a + pp) % 3;
          if (b[bb] > cb[bb] || b[3 + bb] < cb[3 + bb]) covers = 0;
        }
      }
      if (covers) axis = a;
    }
  }
  if (hits != stack_hits) free(hits);
  if (axis < 0) return -1;
  const double pitch = 2.0 * h / n;
  for (int t = 0; t < n; ++t) {
    double p[3] = {c[0], c[1], c[2]};
    p[axis] = c[axis] - h + (t + 0.5) * pitch;
    if (frwo_permittivity_at(s, p, &layers[t]) != 0) return -2;
  }
  int uniform = 1;
  for (int t = 0; t < n; ++t)
    if (!eps_equal(layers[t], layers[0])) uniform = 0;
  if (uniform) axis = 0;
  return axis;
}

/* geometry.cpp:320-349 (classification not needed by the callers here) */
int frwo_build_grid(const frwo_structure *s, const double c[3], double h,
                    int n, double *eps, int32_t *mask) {
  double cb[6] = {c[0] - h, c[1] - h, c[2] - h, c[0] + h, c[1] + h, c[2] + h};
  for (int a = 0; a < 3; ++a)
    if (!(cb[a] >= s->world[a] && cb[3 + a] <= s->world[3 + a])) {
      set_err("build_grid: cube extends outside the world");
      return -1;
    }
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        double p[3];
        voxel_center(c, h, n, i, j, k, p);
        const int idx = (k * n + j) * n + i;
        if (frwo_permittivity_at(s, p, &eps[idx]) != 0) return -1;
        const int ci = frwo_conductor_at(s, p, 0.0);
        if (mask) mask[idx] = ci >= 0 ? s->cond_id[ci] : -1;
        if (ci >= 0 && !mask) {
          set_err("build_grid: cube intersects conductor");
          return -1;
        }
      }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* microwalk.cpp:77-156  absorbing-chain walk                               */

typedef struct {
  /* field: either a materialized grid or a lazily classified structure */
  const double *g_eps;
  const int32_t *g_mask;
  const frwo_structure *s;
  const double *cc; /* cube center */
  double ch;
  int n;
  int conductors;
  frwo_scratch *scr;
} field_t;

struct frwo_scratch {
  int n;
  uint64_t epoch;
  double *eps;
  int32_t *cond;
  uint64_t *stamp;
};

frwo_scratch *frwo_scratch_new(void) {
  return (frwo_scratch *)calloc(1, sizeof(frwo_scratch));
}
void frwo_scratch_free(frwo_scratch *s) {
  if (!s) return;
  free(s->eps);
  free(s->cond);
  free(s->stamp);
  free(s);
}
/* microwalk.cpp:9-21 */
static void scratch_prepare(frwo_scratch *s, int n) {
  if (s->n != n) {
    const size_t tot = (size_t)n * n * n;
    free(s->eps); free(s->cond); free(s->stamp);
    s->eps = calloc(tot, sizeof(double));
    s->cond = malloc(tot * sizeof(int32_t));
    s->stamp = calloc(tot, sizeof(uint64_t));
    s->n = n;
    s->epoch = 0;
  }
  ++s->epoch;
}

/* microwalk.cpp:44-71 LazyField::classify; returns <0 on error */
static int lazy_classify(const field_t *f, int idx, int i, int j, int k) {
  frwo_scratch *scr = f->scr;
  if (scr->stamp[idx] == scr->epoch) return 0;
  double c[3];
  voxel_center(f->cc, f->ch, f->n, i, j, k, c);
  int32_t id = -1;
  if (f->conductors) {
    const int ci = frwo_conductor_at(f->s, c, 0.0);
    if (ci >= 0) id = f->s->cond_id[ci];
  }
  scr->cond[idx] = id;
  if (id >= 0) {
    scr->eps[idx] = 1.0;
  } else if (frwo_permittivity_at(f->s, c, &scr->eps[idx]) != 0) {
    return -1;
  }
  scr->stamp[idx] = scr->epoch;
  return 0;
}

static inline int field_cond(const field_t *f, int idx, int i, int j, int k,
                             int *err) {
  if (f->g_eps) return f->g_mask ? f->g_mask[idx] : -1;
  if (lazy_classify(f, idx, i, j, k)) *err = 1;
  return f->scr->cond[idx];
}
static inline double field_eps(const field_t *f, int idx, int i, int j, int k,
                               int *err) {
  if (f->g_eps) return f->g_eps[idx];
  if (lazy_classify(f, idx, i, j, k)) *err = 1;
  return f->scr->eps[idx];
}

static int walk_lattice(const field_t *f, uint64_t *rng, int step_cap,
                        frwo_exit *e) {
  const int n = f->n;
  if (step_cap <= 0) step_cap = 1000 * n * n;
  int err = 0;
  int node[3] = {(n - 1) / 2, (n - 1) / 2, (n - 1) / 2}; /* sgf.hpp:58-61 */
  int idx = (node[2] * n + node[1]) * n + node[0];
  if (field_cond(f, idx, node[0], node[1], node[2], &err) >= 0) {
    set_err("transit start voxel lies inside a conductor");
    return -3;
  }
  for (int step = 1; step <= step_cap; ++step) {
    /* microwalk.cpp:91-109: alphas in direction order, sum in that order
     * (memoization of the reference is bit-transparent, so recompute) */
    double alpha[6], sum = 0;
    const double ev = field_eps(f, idx, node[0], node[1], node[2], &err);
    for (int d = 0; d < 6; ++d) {
      int nb[3] = {node[0], node[1], node[2]};
      const int a = kDirAxis[d];
      nb[a] += kDirSign[d];
      double al = 1.0;
      if (nb[a] >= 0 && nb[a] < n) {
        const int nidx = (nb[2] * n + nb[1]) * n + nb[0];
        if (field_cond(f, nidx, nb[0], nb[1], nb[2], &err) < 0) {
          const double en = field_eps(f, nidx, nb[0], nb[1], nb[2], &err);
          al = en / (en + ev);
        }
      }
      alpha[d] = al;
      sum += al;
    }
    if (err) return -1;
    /* microwalk.cpp:112-121 */
    const double target = frwo_uniform(rng) * sum;
    double acc = 0;
    int dir = 5;
    for (int d = 0; d < 5; ++d) {
      acc += alpha[d];
      if (target < acc) {
        dir = d;
        break;
      }
    }
    int nb[3] = {node[0], node[1], node[2]};
    const int a = kDirAxis[dir];
    nb[a] += kDirSign[dir];
    if (nb[a] < 0 || nb[a] >= n) { /* microwalk.cpp:126-135 */
      e->kind = 0;
      e->panel = frwo_surface_panel_of(n, node[0], node[1], node[2], dir);
      e->conductor_id = -1;
      frwo_surface_panel_center(f->cc, f->ch, n, e->panel, e->point);
      e->voxel[0] = node[0]; e->voxel[1] = node[1]; e->voxel[2] = node[2];
      e->dir = dir;
      e->steps = step;
      return 0;
    }
    const int nidx = (nb[2] * n + nb[1]) * n + nb[0];
    const int cid = field_cond(f, nidx, nb[0], nb[1], nb[2], &err);
    if (cid >= 0) { /* microwalk.cpp:136-149 */
      e->kind = 1;
      e->panel = -1;
      e->conductor_id = cid;
      voxel_center(f->cc, f->ch, n, node[0], node[1], node[2], e->point);
      e->point[a] += kDirSign[dir] * f->ch / n;
      e->voxel[0] = node[0]; e->voxel[1] = node[1]; e->voxel[2] = node[2];
      e->dir = dir;
      e->steps = step;
      return 0;
    }
    node[0] = nb[0]; node[1] = nb[1]; node[2] = nb[2];
    idx = nidx;
  }
  set_err("microwalk transit exceeded the step cap; the lattice is malformed");
  return -2;
}

int frwo_microwalk_grid(int n, const double *eps, const int32_t *mask,
                        const double c[3], double h, uint64_t *rng,
                        int step_cap, frwo_exit *out) {
  field_t f = {eps, mask, NULL, c, h, n, 0, NULL};
  return walk_lattice(&f, rng, step_cap, out);
}

int frwo_microwalk_lazy(const frwo_structure *s, const double c[3], double h,
                        int n, uint64_t *rng, frwo_scratch *scr, int step_cap,
                        frwo_exit *out) {
  scratch_prepare(scr, n);
  field_t f = {NULL, NULL, s, c, h, n, 0, scr};
  return walk_lattice(&f, rng, step_cap, out);
}

/* microwalk.cpp:206-228 */
int frwo_microwalk_e(const frwo_structure *s, const double center[3],
                     double base_hw, double expansion, int n, uint64_t *rng,
                     frwo_scratch *scr, int step_cap, frwo_exit *out) {
  if (expansion < 1.0) {
    set_err("microwalk_e_transit: expansion must be >= 1");
    return -1;
  }
  const double wall = box_cheb_to_wall(s->world, center);
  const double half = dmin(expansion * base_hw, wall);
  if (!(half > 0)) {
    set_err("microwalk_e_transit: center is on or outside the world wall");
    return -1;
  }
  double cc[3], ch;
  frwo_transit_cube(center, half, n, cc, &ch);
  scratch_prepare(scr, n);
  field_t f = {NULL, NULL, s, cc, ch, n, 1, scr};
  return walk_lattice(&f, rng, step_cap, out);
}

/* batch driver used by the parity tests and the CPU baseline */
typedef struct {
  int n;
  const double *eps;
  const int32_t *mask;
  const double *c;
  double h;
  uint64_t seed, stream0;
  int64_t lo, hi;
  int step_cap;
  int32_t *out_panel, *out_steps;
  uint64_t *hist;
  double ssum, ssq;
  int status;
} grid_job;

static void *grid_worker(void *arg) {
  grid_job *j = (grid_job *)arg;
  for (int64_t t = j->lo; t < j->hi; ++t) {
    uint64_t st = frwo_stream_state(j->seed, j->stream0 + (uint64_t)t);
    frwo_exit e;
    const int rc = frwo_microwalk_grid(j->n, j->eps, j->mask, j->c, j->h, &st,
                                       j->step_cap, &e);
    if (rc) {
      j->status = rc;
      return NULL;
    }
    if (j->out_panel) j->out_panel[t] = e.kind == 0 ? e.panel : -1;
    if (j->out_steps) j->out_steps[t] = e.steps;
    if (j->hist && e.kind == 0) j->hist[e.panel]++;
    j->ssum += e.steps;
    j->ssq += (double)e.steps * e.steps;
  }
  return NULL;
}

int frwo_microwalk_grid_batch(int n, const double *eps, const int32_t *mask,
                              const double c[3], double h, uint64_t seed,
                              uint64_t stream0, int64_t count, int step_cap,
                              int threads, int32_t *out_panel,
                              int32_t *out_steps, uint64_t *hist,
                              double *step_sum, double *step_sumsq) {
  if (threads < 1) threads = 1;
  const int bins = 6 * n * n;
  grid_job *jobs = calloc(threads, sizeof(grid_job));
  pthread_t *tid = calloc(threads, sizeof(pthread_t));
  int64_t lo = 0;
  for (int t = 0; t < threads; ++t) {
    const int64_t hi = lo + count / threads + (t < count % threads);
    grid_job j = {n, eps, mask, c, h, seed, stream0, lo, hi, step_cap,
                  out_panel, out_steps, NULL, 0, 0, 0};
    if (hist) j.hist = calloc(bins, sizeof(uint64_t));
    jobs[t] = j;
    lo = hi;
  }
  for (int t = 0; t < threads; ++t)
    pthread_create(&tid[t], NULL, grid_worker, &jobs[t]);
  int status = 0;
  double ss = 0, sq = 0;
  for (int t = 0; t < threads; ++t) {
    pthread_join(tid[t], NULL);
    if (jobs[t].status) status = jobs[t].status;
    ss += jobs[t].ssum;
    sq += jobs[t].ssq;
    if (hist) {
      for (int b = 0; b < bins; ++b) hist[b] += jobs[t].hist[b];
      free(jobs[t].hist);
    }
  }
  if (step_sum) *step_sum = ss;
  if (step_sumsq) *step_sumsq = sq;
  free(jobs);
  free(tid);
  return status;
}

/* ------------------------------------------------------------------------ */
/* sgf.cpp:57-299  FD system, adjoint PCG solve, kernels, expected steps    */

typedef struct {
  int n, rows;
  double *diag;   /* s_ii diagonal = eps_v * row_sum */
  double *off;    /* [rows][6] s_ii off-diagonals (0 where boundary) */
  double *eps;    /* eps_interior */
  double *rowsum; /* alpha row sums (a_ii diagonal) */
} fdsys;

static void fd_assemble(fdsys *S, int n, const double *eps) {
  const int rows = n * n * n;
  S->n = n;
  S->rows = rows;
  S->diag = malloc(sizeof(double) * rows);
  S->off = calloc((size_t)rows * 6, sizeof(double));
  S->eps = malloc(sizeof(double) * rows);
  S->rowsum = malloc(sizeof(double) * rows);
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        const int idx = (k * n + j) * n + i;
        const double ev = eps[idx];
        S->eps[idx] = ev;
        double rs = 0;
        for (int dir = 0; dir < 6; ++dir) {
          int nb[3] = {i, j, k};
          nb[kDirAxis[dir]] += kDirSign[dir];
          if (nb[0] < 0 || nb[0] >= n || nb[1] < 0 || nb[1] >= n ||
              nb[2] < 0 || nb[2] >= n) {
            rs += 1.0;
            continue;
          }
          const double ei = eps[(nb[2] * n + nb[1]) * n + nb[0]];
          const double alpha = ei / (ei + ev);
          /* sgf.cpp:135-137: bit-symmetric s_ii entry */
          S->off[(size_t)idx * 6 + dir] = -(ev * ei) / (ev + ei);
          rs += alpha;
        }
        S->diag[idx] = ev * rs;
        S->rowsum[idx] = rs;
      }
}

static void fd_free(fdsys *S) {
  free(S->diag); free(S->off); free(S->eps); free(S->rowsum);
}

static void fd_apply(const fdsys *S, const double *x, double *y) {
  const int n = S->n;
  const int stride[6] = {-1, 1, -n, n, -n * n, n * n};
  for (int r = 0; r < S->rows; ++r) {
    double acc = S->diag[r] * x[r];
    const double *o = S->off + (size_t)r * 6;
    for (int d = 0; d < 6; ++d)
      if (o[d] != 0.0) acc += o[d] * x[r + stride[d]];
    y[r] = acc;
  }
}

static double dot(const double *a, const double *b, int m) {
  double s = 0;
  for (int i = 0; i < m; ++i) s += a[i] * b[i];
  return s;
}

/* Eigen::ConjugateGradient + DiagonalPreconditioner, zero initial guess,
 * stop when |r|^2 < tol^2 |b|^2, cap = 20 * rows (sgf.hpp:98-101) */
static int pcg(const fdsys *S, const double *b, double *x) {
  const int m = S->rows;
  const double tol = 1e-10;
  const int maxit = 20 * m;
  double *r = malloc(sizeof(double) * m), *z = malloc(sizeof(double) * m);
  double *p = malloc(sizeof(double) * m), *t = malloc(sizeof(double) * m);
  for (int i = 0; i < m; ++i) {
    x[i] = 0;
    r[i] = b[i];
  }
  const double rhs2 = dot(b, b, m);
  int ok = 1;
  if (rhs2 == 0) goto done;
  const double thresh = tol * tol * rhs2;
  double res2 = dot(r, r, m);
  if (res2 < thresh) goto done;
  for (int i = 0; i < m; ++i) p[i] = r[i] / S->diag[i];
  double absnew = dot(r, p, m);
  ok = 0;
  for (int it = 0; it < maxit; ++it) {
    fd_apply(S, p, t);
    const double alpha = absnew / dot(p, t, m);
    for (int i = 0; i < m; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * t[i];
    }
    res2 = dot(r, r, m);
    if (res2 < thresh) {
      ok = 1;
      break;
    }
    for (int i = 0; i < m; ++i) z[i] = r[i] / S->diag[i];
    const double absold = absnew;
    absnew = dot(r, z, m);
    const double beta = absnew / absold;
    for (int i = 0; i < m; ++i) p[i] = z[i] + beta * p[i];
  }
done:
  free(r); free(z); free(p); free(t);
  return ok ? 0 : -1;
}

/* probs[panel] = (a_ib^T y)[panel]; unmasked: each panel has one row */
static void boundary_gather(int n, const double *y, double *out) {
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        const int idx = (k * n + j) * n + i;
        for (int dir = 0; dir < 6; ++dir) {
          int nb[3] = {i, j, k};
          nb[kDirAxis[dir]] += kDirSign[dir];
          if (nb[0] < 0 || nb[0] >= n || nb[1] < 0 || nb[1] >= n ||
              nb[2] < 0 || nb[2] >= n)
            out[frwo_surface_panel_of(n, i, j, k, dir)] = y[idx];
        }
      }
}

int frwo_solve_sgf(int n, const double *eps, double h, double *probs,
                   double *kernels, double *pitch_out) {
  fdsys S;
  fd_assemble(&S, n, eps);
  const int m = S.rows, panels = 6 * n * n;
  const double pitch = 2.0 * h / n;
  if (pitch_out) *pitch_out = pitch;
  const int c = (n - 1) / 2;
  const int crow = (c * n + c) * n + c;
  double *b = calloc(m, sizeof(double)), *z = malloc(sizeof(double) * m);
  double *pr = malloc(sizeof(double) * panels);
  int rc = 0;
  b[crow] = 1.0;
  if (pcg(&S, b, z)) {
    set_err("transition cube solve failed (PCG did not converge)");
    rc = -1;
    goto out;
  }
  for (int i = 0; i < m; ++i) z[i] *= S.eps[i]; /* adjoint trick */
  boundary_gather(n, z, pr);
  {
    double sum = 0, mn = 1e300;
    for (int q = 0; q < panels; ++q) {
      sum += pr[q];
      mn = dmin(mn, pr[q]);
    }
    if (fabs(sum - 1.0) > 1e-9 || mn < -1e-9) { /* sgf.cpp:249-253 */
      set_err("transition cube solve failed normalization check");
      rc = -2;
      goto out;
    }
  }
  for (int q = 0; q < panels; ++q) probs[q] = dmax(pr[q], 0.0);
  if (kernels) {
    for (int axis = 0; axis < 3; ++axis) {
      double *ker = kernels + (size_t)axis * panels;
      int cp[3] = {c, c, c}, cm[3] = {c, c, c};
      cp[axis] += 1;
      cm[axis] -= 1;
      const int rp = cp[axis] < n ? (cp[2] * n + cp[1]) * n + cp[0] : -1;
      const int rm = cm[axis] >= 0 ? (cm[2] * n + cm[1]) * n + cm[0] : -1;
      memset(b, 0, sizeof(double) * m);
      double denom;
      if (rp >= 0 && rm >= 0) {
        b[rp] = 1.0; b[rm] = -1.0; denom = 2.0 * pitch;
      } else if (rp >= 0) {
        b[rp] = 1.0; b[crow] = -1.0; denom = pitch;
      } else if (rm >= 0) {
        b[crow] = 1.0; b[rm] = -1.0; denom = pitch;
      } else {
        for (int q = 0; q < panels; ++q) ker[q] = 0.0;
        continue;
      }
      if (pcg(&S, b, z)) {
        set_err("kernel solve failed");
        rc = -1;
        goto out;
      }
      for (int i = 0; i < m; ++i) z[i] *= S.eps[i];
      boundary_gather(n, z, pr);
      for (int q = 0; q < panels; ++q) ker[q] = pr[q] / denom;
    }
  }
out:
  free(b); free(z); free(pr);
  fd_free(&S);
  return rc;
}

double frwo_expected_steps(int n, const double *eps) {
  fdsys S;
  fd_assemble(&S, n, eps);
  const int m = S.rows;
  double *b = malloc(sizeof(double) * m), *t = malloc(sizeof(double) * m);
  for (int i = 0; i < m; ++i) b[i] = S.eps[i] * S.rowsum[i];
  double out = NAN;
  if (pcg(&S, b, t) == 0) {
    const int c = (n - 1) / 2;
    out = t[(c * n + c) * n + c];
  }
  free(b); free(t);
  fd_free(&S);
  return out;
}

/* sgf.cpp:301-308: upper_bound on the inclusive CDF, clamp to last */
int frwo_sample_panel(const double *cdf, int count, double u) {
  const double target = u * cdf[count - 1];
  int lo = 0, hi = count;
  while (lo < hi) {
    const int mid = lo + (hi - lo) / 2;
    if (target < cdf[mid]) hi = mid; else lo = mid + 1;
  }
  return lo == count ? count - 1 : lo;
}

/* sgf_cache.cpp:13-18 */
double frwo_round_sig(double x, int digits) {
  if (x == 0 || !isfinite(x)) return x;
  const double e10 = floor(log10(fabs(x)));
  const double mag = pow(10.0, digits - 1 - e10);
  return round(x * mag) / mag;
}

/* ------------------------------------------------------------------------ */
/* sgf_cache.cpp:29-153  concurrent memo of canonical stratified SGFs       */

typedef struct {
  int n, axis;
  double *layers;
  uint64_t hash;
  double pitch;
  double *probs, *cdf, *kern; /* kern: 3 x 6n^2 */
} sgf_entry;

typedef struct {
  pthread_rwlock_t mu;
  sgf_entry **slots;
  size_t cap, size;
  uint64_t hits, misses;
  pthread_mutex_t stat_mu;
} sgf_cache;

static uint64_t key_hash(int n, int axis, const double *layers) {
  uint64_t h = frwo_mix(((uint64_t)n << 8) ^ (uint64_t)axis);
  for (int t = 0; t < n; ++t) {
    uint64_t bits;
    memcpy(&bits, &layers[t], 8);
    h = frwo_mix(h ^ bits);
  }
  return h;
}

static sgf_entry *cache_find(sgf_cache *C, int n, int axis,
                             const double *layers, uint64_t h) {
  if (!C->cap) return NULL;
  for (size_t i = h & (C->cap - 1);; i = (i + 1) & (C->cap - 1)) {
    sgf_entry *e = C->slots[i];
    if (!e) return NULL;
    if (e->hash == h && e->n == n && e->axis == axis &&
        !memcmp(e->layers, layers, sizeof(double) * n))
      return e;
  }
}

static void cache_insert_locked(sgf_cache *C, sgf_entry *e) {
  if ((C->size + 1) * 2 > C->cap) {
    size_t ncap = C->cap ? C->cap * 2 : 64;
    sgf_entry **ns = calloc(ncap, sizeof(sgf_entry *));
    for (size_t i = 0; i < C->cap; ++i)
      if (C->slots[i]) {
        size_t j = C->slots[i]->hash & (ncap - 1);
        while (ns[j]) j = (j + 1) & (ncap - 1);
        ns[j] = C->slots[i];
      }
    free(C->slots);
    C->slots = ns;
    C->cap = ncap;
  }
  size_t j = e->hash & (C->cap - 1);
  while (C->slots[j]) j = (j + 1) & (C->cap - 1);
  C->slots[j] = e;
  C->size++;
}

static void cache_destroy(sgf_cache *C) {
  for (size_t i = 0; i < C->cap; ++i)
    if (C->slots[i]) {
      sgf_entry *e = C->slots[i];
      free(e->layers); free(e->probs); free(e->cdf); free(e->kern); free(e);
    }
  free(C->slots);
  pthread_rwlock_destroy(&C->mu);
  pthread_mutex_destroy(&C->stat_mu);
}

/* profile_key (sgf_cache.cpp:29-51) then get (sgf_cache.cpp:107-131) */
static sgf_entry *cache_get(sgf_cache *C, int n, int axis,
                            const double *raw_layers) {
  double layers[256];
  for (int t = 0; t < n; ++t) layers[t] = frwo_round_sig(raw_layers[t], 6);
  int uniform = 1;
  for (int t = 0; t < n; ++t) uniform = uniform && layers[t] == layers[0];
  if (uniform) axis = 0;
  const uint64_t h = key_hash(n, axis, layers);
  pthread_rwlock_rdlock(&C->mu);
  sgf_entry *e = cache_find(C, n, axis, layers, h);
  pthread_rwlock_unlock(&C->mu);
  pthread_mutex_lock(&C->stat_mu);
  if (e) C->hits++; else C->misses++;
  pthread_mutex_unlock(&C->stat_mu);
  if (e) return e;
  /* canonical_grid (sgf_cache.cpp:78-96): unit pitch, half width n/2 */
  const size_t nv = (size_t)n * n * n;
  double *eps = malloc(sizeof(double) * nv);
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        const int v[3] = {i, j, k};
        eps[(k * n + j) * n + i] = layers[v[axis]];
      }
  const int panels = 6 * n * n;
  sgf_entry *ne = calloc(1, sizeof(sgf_entry));
  ne->n = n;
  ne->axis = axis;
  ne->hash = h;
  ne->layers = malloc(sizeof(double) * n);
  memcpy(ne->layers, layers, sizeof(double) * n);
  ne->probs = malloc(sizeof(double) * panels);
  ne->cdf = malloc(sizeof(double) * panels);
  ne->kern = malloc(sizeof(double) * 3 * panels);
  const int rc =
      frwo_solve_sgf(n, eps, n / 2.0, ne->probs, ne->kern, &ne->pitch);
  free(eps);
  if (rc) {
    free(ne->layers); free(ne->probs); free(ne->cdf); free(ne->kern); free(ne);
    return NULL;
  }
  double run = 0;
  for (int q = 0; q < panels; ++q) {
    run += ne->probs[q];
    ne->cdf[q] = run;
  }
  pthread_rwlock_wrlock(&C->mu);
  sgf_entry *ex = cache_find(C, n, axis, layers, h);
  if (ex) { /* lost the race: first result wins */
    pthread_rwlock_unlock(&C->mu);
    free(ne->layers); free(ne->probs); free(ne->cdf); free(ne->kern); free(ne);
    return ex;
  }
  cache_insert_locked(C, ne);
  pthread_rwlock_unlock(&C->mu);
  return ne;
}

/* ------------------------------------------------------------------------ */
/* engine.cpp  walk engine                                                  */

#define EPS0 8.8541878128e-12 /* constants.hpp:5 */
#define M_PER_NM 1e-9         /* constants.hpp:6 */

void frwo_config_default(frwo_config *c) { /* engine.hpp:28-43 */
  c->grid_n = 24;
  c->expansion = 5.0;
  c->mode = FRWO_HYBRID_MWE;
  c->rel_std_tol = 0.01;
  c->min_walks = 4096;
  c->max_walks = 4000000;
  c->batch = 1024;
  c->seed = 1;
  c->snap_tol = 1e-4;
  c->hop_cap = 10000;
  c->gaussian_gap_fraction = 0.5;
  c->world_margin = 5.0;
  c->all_couplings_rule = 0;
}

typedef struct {
  const frwo_structure *s;
  frwo_config cfg;
  double gbox[6];
  double area_m2;
  double face_cdf[6];
  double snap;
  int master_slot, ground_slot;
  sgf_cache cache;
} engine_t;

typedef struct {
  uint64_t first[4], sub[4];
  uint64_t resampled;
  uint64_t mw_steps;
} wstats;

/* engine.cpp:84-124 */
static int gaussian_surface(engine_t *E) {
  const frwo_structure *s = E->s;
  int m = -1;
  for (int c = 0; c < s->n_cond; ++c)
    if (s->cond_id[c] == s->master_id) { m = c; break; }
  if (m < 0) {
    set_err("master conductor not found");
    return -1;
  }
  const double *mb = s->cond_box + 6 * m;
  double gap = INFINITY;
  for (int ax = 0; ax < 3; ++ax) {
    gap = dmin(gap, mb[ax] - s->world[ax]);
    gap = dmin(gap, s->world[3 + ax] - mb[3 + ax]);
  }
  for (int c = 0; c < s->n_cond; ++c) {
    if (s->cond_id[c] == s->master_id) continue;
    const double *cb = s->cond_box + 6 * c;
    double g = 0; /* engine.cpp:27-35 box_gap */
    for (int ax = 0; ax < 3; ++ax)
      g = dmax(g, dmax(mb[ax] - cb[3 + ax], cb[ax] - mb[3 + ax]));
    gap = dmin(gap, dmax(g, 0.0));
  }
  if (!(gap > 0.0)) {
    set_err("master touches another conductor or the wall");
    return -1;
  }
  const double inflate = E->cfg.gaussian_gap_fraction * gap;
  for (int ax = 0; ax < 3; ++ax) {
    E->gbox[ax] = mb[ax] - inflate;
    E->gbox[3 + ax] = mb[3 + ax] + inflate;
  }
  const double ex = E->gbox[3] - E->gbox[0];
  const double ey = E->gbox[4] - E->gbox[1];
  const double ez = E->gbox[5] - E->gbox[2];
  const double f[6] = {ey * ez, ey * ez, ex * ez, ex * ez, ex * ey, ex * ey};
  double total = 0;
  for (int i = 0; i < 6; ++i) total += f[i];
  double acc = 0;
  for (int i = 0; i < 6; ++i) {
    acc += f[i] / total;
    E->face_cdf[i] = acc;
  }
  E->face_cdf[5] = 1.0;
  E->area_m2 = total * M_PER_NM * M_PER_NM;
  E->master_slot = m;
  E->ground_slot = s->n_cond;
  /* engine.cpp:186-187 */
  double he = 0;
  for (int ax = 0; ax < 3; ++ax)
    he = dmax(he, (E->gbox[3 + ax] - E->gbox[ax]) / 2);
  E->snap = E->cfg.snap_tol * he;
  return 0;
}

/* engine.cpp:126-148 */
static void sample_gaussian(const engine_t *E, uint64_t *rng, double p[3],
                            int *axis, int *sign) {
  const double u = frwo_uniform(rng);
  int face = 5;
  for (int f = 0; f < 5; ++f)
    if (u < E->face_cdf[f]) { face = f; break; }
  const int a = kDirAxis[face];
  const int b1 = a == 0 ? 1 : 0;
  const int b2 = a == 2 ? 1 : 2;
  *axis = a;
  *sign = kDirSign[face];
  p[a] = *sign < 0 ? E->gbox[a] : E->gbox[3 + a];
  p[b1] = E->gbox[b1] + frwo_uniform(rng) * (E->gbox[3 + b1] - E->gbox[b1]);
  p[b2] = E->gbox[b2] + frwo_uniform(rng) * (E->gbox[3 + b2] - E->gbox[b2]);
}

/* engine.cpp:201-288; returns 1 ok, 0 degenerate (redraw), <0 error */
static int first_transition(engine_t *E, const double gp[3], int gaxis,
                            int gsign, uint64_t *rng, wstats *st,
                            double out_p[3], double *weight) {
  const frwo_structure *s = E->s;
  if (frwo_conductor_at(s, gp, E->snap) >= 0) return 0;
  double fh;
  if (frwo_max_free_cube(s, gp, &fh, NULL)) return -1;
  if (!(fh > E->snap)) return 0;
  const int n = E->cfg.grid_n;
  double cc[3], ch;
  frwo_transit_cube(gp, fh, n, cc, &ch);
  double layers[256];
  int axis = frwo_stratified_profile(s, cc, ch, n, layers);
  if (axis == -2) return -1;
  int branch = 0;
  if (axis < 0) {
    for (int i = 19; i >= 6; --i) {
      double c2[3], h2;
      frwo_transit_cube(gp, 0.05 * i * fh, n, c2, &h2);
      axis = frwo_stratified_profile(s, c2, h2, n, layers);
      if (axis == -2) return -1;
      if (axis >= 0) {
        memcpy(cc, c2, sizeof cc);
        ch = h2;
        branch = 1;
        break;
      }
    }
  }
  if (axis < 0) {
    const size_t nv = (size_t)n * n * n;
    double *eps = malloc(sizeof(double) * nv);
    if (frwo_build_grid(s, cc, ch, n, eps, NULL)) {
      free(eps);
      return -1;
    }
    double slice[3][256];
    memset(slice, 0, sizeof slice);
    size_t idx = 0;
    for (int k = 0; k < n; ++k)
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i, ++idx) {
          const double e = eps[idx];
          slice[0][i] += e;
          slice[1][j] += e;
          slice[2][k] += e;
        }
    free(eps);
    int best = 0;
    double bvar = -1.0;
    for (int ax = 0; ax < 3; ++ax) {
      double mean = 0;
      for (int t = 0; t < n; ++t) {
        slice[ax][t] /= (double)n * n;
        mean += slice[ax][t];
      }
      mean /= n;
      double var = 0;
      for (int t = 0; t < n; ++t)
        var += (slice[ax][t] - mean) * (slice[ax][t] - mean);
      if (var > bvar) {
        bvar = var;
        best = ax;
      }
    }
    axis = best;
    memcpy(layers, slice[best], sizeof(double) * n);
    branch = 2;
    int uni = 1;
    for (int t = 0; t < n; ++t)
      if (frwo_round_sig(layers[t], 6) != frwo_round_sig(layers[0], 6))
        uni = 0;
    if (uni) branch = 3;
  }
  st->first[branch]++;
  sgf_entry *g = cache_get(&E->cache, n, axis, layers);
  if (!g) return -1;
  const int panels = 6 * n * n;
  const int panel = frwo_sample_panel(g->cdf, panels, frwo_uniform(rng));
  const double pitch_nm = 2.0 * ch / n;
  const double kern_per_m =
      g->kern[(size_t)gaxis * panels + panel] * (g->pitch / pitch_nm) /
      M_PER_NM;
  double eps_r;
  if (frwo_permittivity_at(s, gp, &eps_r)) return -1;
  frwo_surface_panel_center(cc, ch, n, panel, out_p);
  *weight = -E->area_m2 * EPS0 * eps_r * gsign * kern_per_m / g->probs[panel];
  return 1;
}

/* engine.cpp:290-350; returns 0 continue, 1 terminate(cond), 2 ground,
 * <0 error */
static int transition(engine_t *E, double p[3], uint64_t *rng,
                      frwo_scratch *scr, wstats *st, int *cond_index) {
  const frwo_structure *s = E->s;
  const int ci = frwo_conductor_at(s, p, E->snap);
  if (ci >= 0) {
    *cond_index = ci;
    return 1;
  }
  if (box_cheb_to_wall(s->world, p) <= E->snap) return 2;
  double fh;
  if (frwo_max_free_cube(s, p, &fh, NULL)) return -1;
  const int n = E->cfg.grid_n;
  double cc[3], ch;
  frwo_transit_cube(p, fh, n, cc, &ch);
  double layers[256];
  const int axis = frwo_stratified_profile(s, cc, ch, n, layers);
  if (axis == -2) return -1;
  const int panels = 6 * n * n;
  if (axis >= 0) {
    st->sub[0]++;
    sgf_entry *g = cache_get(&E->cache, n, axis, layers);
    if (!g) return -1;
    const int panel = frwo_sample_panel(g->cdf, panels, frwo_uniform(rng));
    frwo_surface_panel_center(cc, ch, n, panel, p);
    return 0;
  }
  frwo_exit e;
  switch (E->cfg.mode) {
    case FRWO_FDM: {
      st->sub[3]++;
      const size_t nv = (size_t)n * n * n;
      double *eps = malloc(sizeof(double) * nv);
      double *pr = malloc(sizeof(double) * panels);
      int rc = frwo_build_grid(s, cc, ch, n, eps, NULL);
      if (!rc) rc = frwo_solve_sgf(n, eps, ch, pr, NULL, NULL);
      if (!rc) {
        double run = 0;
        for (int q = 0; q < panels; ++q) { run += pr[q]; pr[q] = run; }
        const int panel = frwo_sample_panel(pr, panels, frwo_uniform(rng));
        frwo_surface_panel_center(cc, ch, n, panel, p);
      }
      free(eps); free(pr);
      return rc ? -1 : 0;
    }
    case FRWO_MW:
    case FRWO_HYBRID_MW: {
      st->sub[1]++;
      const int rc = frwo_microwalk_lazy(s, cc, ch, n, rng, scr, 0, &e);
      if (rc) return -1;
      st->mw_steps += e.steps;
      memcpy(p, e.point, sizeof(double) * 3);
      return 0;
    }
    default: {
      st->sub[2]++;
      int rc = frwo_microwalk_e(s, p, fh, E->cfg.expansion, n, rng, scr, 0,
                                &e);
      if (rc == -3) { /* EngulfedStart: walk the plain cube instead */
        rc = frwo_microwalk_lazy(s, cc, ch, n, rng, scr, 0, &e);
        if (rc) return -1;
        st->mw_steps += e.steps;
        memcpy(p, e.point, sizeof(double) * 3);
        return 0;
      }
      if (rc) return -1;
      st->mw_steps += e.steps;
      if (e.kind == 1) {
        for (int c = 0; c < s->n_cond; ++c)
          if (s->cond_id[c] == e.conductor_id) *cond_index = c;
        memcpy(p, e.point, sizeof(double) * 3);
        return 1;
      }
      memcpy(p, e.point, sizeof(double) * 3);
      return 0;
    }
  }
}

/* engine.cpp:352-376 */
static int run_walk(engine_t *E, uint64_t walk, frwo_scratch *scr,
                    wstats *st, int32_t *slot, double *weight,
                    uint8_t *aborted) {
  uint64_t rng = frwo_stream_state(E->cfg.seed, walk);
  double p[3], w = 0;
  int ok = 0;
  for (int attempt = 0; attempt < 100 && !ok; ++attempt) {
    double gp[3];
    int ga, gs;
    sample_gaussian(E, &rng, gp, &ga, &gs);
    const int rc = first_transition(E, gp, ga, gs, &rng, st, p, &w);
    if (rc < 0) return -1;
    if (rc == 0) st->resampled++;
    ok = rc;
  }
  if (!ok) {
    *slot = E->ground_slot; *weight = 0.0; *aborted = 1;
    return 0;
  }
  for (int64_t hop = 0; hop < E->cfg.hop_cap; ++hop) {
    int ci = -1;
    const int rc = transition(E, p, &rng, scr, st, &ci);
    if (rc < 0) return -1;
    if (rc == 1) {
      *slot = ci; *weight = w; *aborted = 0;
      return 0;
    }
    if (rc == 2) {
      *slot = E->ground_slot; *weight = w; *aborted = 0;
      return 0;
    }
  }
  *slot = E->ground_slot; *weight = w; *aborted = 1;
  return 0;
}

typedef struct {
  engine_t *E;
  uint64_t w0;
  int64_t lo, hi;
  int32_t *slot;
  double *weight;
  uint8_t *aborted;
  wstats st;
  int status;
  char err[512];
} walk_job;

static void *walk_worker(void *arg) {
  walk_job *j = (walk_job *)arg;
  frwo_scratch *scr = frwo_scratch_new();
  for (int64_t i = j->lo; i < j->hi; ++i)
    if (run_walk(j->E, j->w0 + i, scr, &j->st, &j->slot[i], &j->weight[i],
                 &j->aborted[i])) {
      j->status = -1;
      snprintf(j->err, sizeof j->err, "%s", g_err);
      break;
    }
  frwo_scratch_free(scr);
  return NULL;
}

static int run_range(engine_t *E, uint64_t w0, int64_t count, int threads,
                     int32_t *slot, double *weight, uint8_t *aborted,
                     wstats *acc) {
  if (threads < 1) threads = 1;
  walk_job *jobs = calloc(threads, sizeof(walk_job));
  pthread_t *tid = calloc(threads, sizeof(pthread_t));
  int64_t lo = 0;
  for (int t = 0; t < threads; ++t) {
    const int64_t hi = lo + count / threads + (t < count % threads);
    jobs[t].E = E; jobs[t].w0 = w0; jobs[t].lo = lo; jobs[t].hi = hi;
    jobs[t].slot = slot; jobs[t].weight = weight; jobs[t].aborted = aborted;
    lo = hi;
  }
  if (threads == 1) {
    walk_worker(&jobs[0]);
  } else {
    for (int t = 0; t < threads; ++t)
      pthread_create(&tid[t], NULL, walk_worker, &jobs[t]);
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  }
  int status = 0;
  for (int t = 0; t < threads; ++t) {
    if (jobs[t].status) {
      status = -1;
      set_err(jobs[t].err);
    }
    for (int b = 0; b < 4; ++b) {
      acc->first[b] += jobs[t].st.first[b];
      acc->sub[b] += jobs[t].st.sub[b];
    }
    acc->resampled += jobs[t].st.resampled;
    acc->mw_steps += jobs[t].st.mw_steps;
  }
  free(jobs);
  free(tid);
  return status;
}

static int engine_init(engine_t *E, const frwo_structure *s,
                       const frwo_config *c) {
  memset(E, 0, sizeof *E);
  E->s = s;
  E->cfg = *c;
  if (c->grid_n < 2 || c->grid_n > 256) {
    set_err("grid_n must be in [2, 256]");
    return -1;
  }
  pthread_rwlock_init(&E->cache.mu, NULL);
  pthread_mutex_init(&E->cache.stat_mu, NULL);
  return gaussian_surface(E);
}

int frwo_run_walks(const frwo_structure *s, const frwo_config *c, uint64_t w0,
                   int64_t count, int threads, int32_t *slot, double *weight,
                   uint8_t *aborted) {
  engine_t E;
  if (engine_init(&E, s, c)) return -1;
  wstats acc;
  memset(&acc, 0, sizeof acc);
  const int rc = run_range(&E, w0, count, threads, slot, weight, aborted, &acc);
  cache_destroy(&E.cache);
  return rc;
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

/* engine.cpp:378-507 */
int frwo_extract(const frwo_structure *s, const frwo_config *c, int threads,
                 frwo_result *res) {
  const double t0 = now_s();
  engine_t E;
  if (engine_init(&E, s, c)) return -1;
  const int nslots = s->n_cond + 1;
  for (int k = 0; k < nslots; ++k) {
    res->sum[k] = res->sumsq[k] = 0;
    res->landed[k] = 0;
  }
  wstats acc;
  memset(&acc, 0, sizeof acc);
  uint64_t walks = 0, aborted = 0;
  int converged = 0, status = 0;
  const int64_t B = c->batch;
  int32_t *slot = malloc(sizeof(int32_t) * B);
  double *weight = malloc(sizeof(double) * B);
  uint8_t *ab = malloc(B);
  while (walks < (uint64_t)c->max_walks) {
    const int64_t bsz = (int64_t)((uint64_t)c->max_walks - walks) < B
                            ? (int64_t)((uint64_t)c->max_walks - walks)
                            : B;
    if (run_range(&E, walks, bsz, threads, slot, weight, ab, &acc)) {
      status = -1;
      break;
    }
    for (int64_t i = 0; i < bsz; ++i) { /* fold in walk order */
      res->sum[slot[i]] += weight[i];
      res->sumsq[slot[i]] += weight[i] * weight[i];
      res->landed[slot[i]]++;
      aborted += ab[i];
    }
    walks += bsz;
    if (walks >= (uint64_t)c->min_walks) {
      /* engine.cpp:388-420 */
      const double w = (double)walks;
      double mean[1024 + 1], se[1024 + 1];
      for (int k = 0; k < nslots && k <= 1024; ++k) {
        mean[k] = res->sum[k] / w;
        double v = 0;
        if (walks > 1) {
          v = dmax(0.0, (res->sumsq[k] - res->sum[k] * res->sum[k] / w) /
                            (w - 1));
          se[k] = sqrt(v / w);
        } else {
          se[k] = 0;
        }
      }
      const int m = E.master_slot;
      int conv = 0;
      if (mean[m] > 0 && !(se[m] > c->rel_std_tol * mean[m])) {
        if (c->all_couplings_rule) {
          conv = 1;
          for (int k = 0; k < s->n_cond; ++k)
            if (k != m && se[k] > c->rel_std_tol * fabs(mean[k])) conv = 0;
        } else {
          int big = nslots;
          double big_abs = 0;
          for (int k = 0; k < nslots; ++k) {
            if (k == m) continue;
            const double a = fabs(res->sum[k] / w);
            if (a > big_abs) { big_abs = a; big = k; }
          }
          conv = big == nslots ? 1 : se[big] <= c->rel_std_tol * fabs(mean[big]);
        }
      }
      if (conv) {
        converged = 1;
        break;
      }
    }
  }
  free(slot); free(weight); free(ab);
  const double w = (double)walks;
  for (int k = 0; k < nslots; ++k) {
    res->value[k] = res->sum[k] / w;
    double se = 0;
    if (walks > 1) {
      const double v = dmax(
          0.0, (res->sumsq[k] - res->sum[k] * res->sum[k] / w) / (w - 1));
      se = sqrt(v / w);
    }
    res->std_err[k] = se;
  }
  res->walks = walks;
  res->converged = converged;
  res->aborted = aborted;
  res->resampled = acc.resampled;
  memcpy(res->first, acc.first, sizeof acc.first);
  memcpy(res->sub, acc.sub, sizeof acc.sub);
  res->cache_hits = E.cache.hits;
  res->cache_misses = E.cache.misses;
  res->mw_steps = acc.mw_steps;
  cache_destroy(&E.cache);
  res->t_total_seconds = now_s() - t0;
  return status;
}
