/* oracle/sw2d_ref.c — TEST INFRASTRUCTURE ONLY (the parity oracle).
 *
 * A plain, slow, single-threaded C11 implementation of one time step of the
 * 2-D shallow water model (2DSW) that arXiv 1711.04471 auto-parallelises:
 * "a time loop which calls two subroutines, a predictor (dyn) and a
 * first-order Shapiro filter (shapiro), before updating the velocity"
 * (§6.2).  The paper prints no equations; the scheme is the
 * cited textbook's (Kaempf 2009) C-grid forward-backward scheme
 * as read in DESIGN.md "Readings" R1-R17.
 *
 * Who may use it: tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg.  The product path never links it.
 * It shares no code with paper_1711_04471_b200/ (no header, no helper, no
 * constant generator).
 *
 * Arithmetic: IEEE binary32, round-to-nearest-even, every operation rounded
 * separately (build with -std=c11 -O2 -ffp-contract=off -fno-fast-math so no
 * FMA contraction and no reassociation), in the order written in DESIGN.md
 * §"Oracle step" — which is the order written below, statement by statement.
 * Every read inside a step is of the step-n state (map / Jacobi semantics: the
 * paper's kernels are maps).
 *
 * Pins (tests/test_oracle_pins.py): 3x3 and 1x4 hand-computed golden steps
 * (tests/golden/), lake at rest (bitwise), volume conservation (1e-6),
 * mirror symmetry (bitwise), linear wave speed sqrt(gH) (2%), Merian seiche
 * period (1%), g=0 Shapiro eigen-decay (closed form, 1e-5), Thacker planar
 * oscillation period (2%), reductions on closed-form states.
 * The blocked-face velocity rule (R4) and the operation order (R12) are
 * "parity unpinned" by the paper: pinned only by the DESIGN.md reading.
 */
#include "sw2d_ref.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* Halo'd working grid: (ny+2) x (nx+2), interior j = 1..ny, k = 1..nx. */
#define AT(a, j, k) (a)[(size_t)(j) * (size_t)(nx + 2) + (size_t)(k)]

/* Upwind volume flux through a face with velocity s between a left/lower cell
 * of depth hL and a right/upper cell of depth hR (reading R3, upwind depth). */
static float flux(float s, float hL, float hR) {
  if (s > 0.0f) return s * hL;
  if (s < 0.0f) return s * hR;
  return 0.0f;
}

/* sel(m, x) = m ? x : 0 — the textbook's wet*etan, as a select (R12). */
static float sel(int m, float x) { return m ? x : 0.0f; }

typedef struct {
  float cgx, cgy, cx, cy, q, hmin;
} coeffs;

/* Coefficients, once, on the host: double then one rounding (R12). */
static coeffs make_coeffs(const sw2d_ref_params* p) {
  coeffs c;
  double t = (double)p->dt * (double)p->g;
  c.cgx = (float)(-(t / (double)p->dx));
  c.cgy = (float)(-(t / (double)p->dy));
  c.cx = (float)((double)p->dt / (double)p->dx);
  c.cy = (float)((double)p->dt / (double)p->dy);
  c.q = 0.25f * p->eps;
  c.hmin = p->hmin;
  return c;
}

typedef struct {
  int64_t nx, ny;
  float *H0, *E, *U, *V, *h, *un, *vn, *etan;
  unsigned char* w;
} grid;

static void grid_free(grid* G) {
  free(G->H0); free(G->E); free(G->U); free(G->V); free(G->h);
  free(G->un); free(G->vn); free(G->etan); free(G->w);
}

static int grid_alloc(grid* G, int64_t nx, int64_t ny) {
  size_t n = (size_t)(nx + 2) * (size_t)(ny + 2);
  memset(G, 0, sizeof(*G));
  G->nx = nx; G->ny = ny;
  G->H0 = calloc(n, sizeof(float)); G->E = calloc(n, sizeof(float));
  G->U = calloc(n, sizeof(float));  G->V = calloc(n, sizeof(float));
  G->h = calloc(n, sizeof(float));  G->un = calloc(n, sizeof(float));
  G->vn = calloc(n, sizeof(float)); G->etan = calloc(n, sizeof(float));
  G->w = calloc(n, 1);
  if (!G->H0 || !G->E || !G->U || !G->V || !G->h || !G->un || !G->vn ||
      !G->etan || !G->w) {
    grid_free(G);
    return -1;
  }
  return 0;
}

/* One time step (rows a1..a5). */
static void step(grid* G, const coeffs* c) {
  const int64_t nx = G->nx, ny = G->ny;
  int64_t j, k;

  /* a1: derived state (textbook update of h and wet).  Halo ring: w = 0. */
  for (j = 0; j <= ny + 1; j++)
    for (k = 0; k <= nx + 1; k++) {
      if (j >= 1 && j <= ny && k >= 1 && k <= nx) {
        AT(G->h, j, k) = AT(G->H0, j, k) + AT(G->E, j, k);
        AT(G->w, j, k) = !(AT(G->h, j, k) < c->hmin);
      } else {
        AT(G->h, j, k) = 0.0f;
        AT(G->w, j, k) = 0;
      }
    }

  /* a2: momentum predictor (dyn, part 1) with the wet/dry face rule (R4):
   * a face carries flow if its upstream cell is wet; a blocked face gets 0.
   * CLOSED walls (R5): east faces k = nx, north faces j = ny, and the west
   * (k = 0) / south (j = 0) faces are 0. */
  for (j = 1; j <= ny; j++)
    for (k = 1; k <= nx; k++) {
      if (k == nx) {
        AT(G->un, j, k) = 0.0f;
      } else {
        float du = c->cgx * (AT(G->E, j, k + 1) - AT(G->E, j, k));
        int wc = AT(G->w, j, k), we = AT(G->w, j, k + 1);
        int flow = wc ? (we || du > 0.0f) : (we && du < 0.0f);
        AT(G->un, j, k) = flow ? AT(G->U, j, k) + du : 0.0f;
      }
      if (j == ny) {
        AT(G->vn, j, k) = 0.0f;
      } else {
        float dv = c->cgy * (AT(G->E, j + 1, k) - AT(G->E, j, k));
        int wc = AT(G->w, j, k), wn = AT(G->w, j + 1, k);
        int flow = wc ? (wn || dv > 0.0f) : (wn && dv < 0.0f);
        AT(G->vn, j, k) = flow ? AT(G->V, j, k) + dv : 0.0f;
      }
    }
  for (j = 0; j <= ny + 1; j++) { AT(G->un, j, 0) = 0.0f; }
  for (k = 0; k <= nx + 1; k++) { AT(G->vn, 0, k) = 0.0f; }

  /* a3: sea-level predictor (dyn, part 2): upwind volume-flux divergence. */
  for (j = 1; j <= ny; j++)
    for (k = 1; k <= nx; k++) {
      float hc = AT(G->h, j, k);
      float fe = flux(AT(G->un, j, k), hc, AT(G->h, j, k + 1));
      float fw = flux(AT(G->un, j, k - 1), AT(G->h, j, k - 1), hc);
      float fn = flux(AT(G->vn, j, k), hc, AT(G->h, j + 1, k));
      float fs = flux(AT(G->vn, j - 1, k), AT(G->h, j - 1, k), hc);
      AT(G->etan, j, k) =
          (AT(G->E, j, k) - c->cx * (fe - fw)) - c->cy * (fn - fs);
    }

  /* a4: first-order Shapiro filter, wet-masked (shapiro).
   * a5: state commit eta <- eta', u <- un, v <- vn ("updating the velocity",
   * PAPER.md:372).  Written into E after all of etan exists (map semantics). */
  for (j = 1; j <= ny; j++)
    for (k = 1; k <= nx; k++) {
      float en = AT(G->etan, j, k);
      if (AT(G->w, j, k)) {
        int wE = AT(G->w, j, k + 1), wW = AT(G->w, j, k - 1);
        int wN = AT(G->w, j + 1, k), wS = AT(G->w, j - 1, k);
        float s = (float)(wE + wW + wN + wS);
        float t1 = (1.0f - c->q * s) * en;
        float t2 = c->q * (sel(wE, AT(G->etan, j, k + 1)) +
                           sel(wW, AT(G->etan, j, k - 1)));
        float t3 = c->q * (sel(wN, AT(G->etan, j + 1, k)) +
                           sel(wS, AT(G->etan, j - 1, k)));
        AT(G->E, j, k) = (t1 + t2) + t3;
      } else {
        AT(G->E, j, k) = en;
      }
    }
  for (j = 1; j <= ny; j++)
    for (k = 1; k <= nx; k++) {
      AT(G->U, j, k) = AT(G->un, j, k);
      AT(G->V, j, k) = AT(G->vn, j, k);
    }
}

/* Neumaier-compensated sum accumulator. */
typedef struct { double s, c; } nsum;
static void nadd(nsum* a, double x) {
  double t = a->s + x;
  if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x;
  else a->c += (x - t) + a->s;
  a->s = t;
}

/* a6: diagnostics of the state held in G (reading R16). */
static void reduce(const grid* G, const sw2d_ref_params* p, double* out) {
  const int64_t nx = G->nx, ny = G->ny;
  nsum vol = {0, 0}, se = {0, 0};
  float mx = -INFINITY, mn = INFINITY, mu = 0.0f, mv = 0.0f;
  int64_t wet = 0, j, k;
  for (j = 1; j <= ny; j++)
    for (k = 1; k <= nx; k++) {
      float e = AT(G->E, j, k), h0 = AT(G->H0, j, k);
      nadd(&vol, (double)h0 + (double)e);
      nadd(&se, (double)e);
      if (e > mx) mx = e;
      if (e < mn) mn = e;
      if (fabsf(AT(G->U, j, k)) > mu) mu = fabsf(AT(G->U, j, k));
      if (fabsf(AT(G->V, j, k)) > mv) mv = fabsf(AT(G->V, j, k));
      wet += !(h0 + e < p->hmin);
    }
  out[SW2D_REF_VOLUME] = (double)p->dx * (double)p->dy * (vol.s + vol.c);
  out[SW2D_REF_SUM_ETA] = se.s + se.c;
  out[SW2D_REF_MAX_ETA] = mx;
  out[SW2D_REF_MIN_ETA] = mn;
  out[SW2D_REF_MAX_ABS_U] = mu;
  out[SW2D_REF_MAX_ABS_V] = mv;
  out[SW2D_REF_WET_COUNT] = (double)wet;
}

static int bad(const sw2d_ref_params* p, int64_t nx, int64_t ny) {
  if (!p || nx < 1 || ny < 1) return 1;
  if (!(p->dx > 0.0f) || !(p->dy > 0.0f) || !(p->dt > 0.0f)) return 1;
  if (!(p->g >= 0.0f) || !(p->eps >= 0.0f && p->eps <= 1.0f)) return 1;
  if (!(p->hmin >= 0.0f)) return 1;
  return 0;
}

/* Copy host arrays into the halo'd grid; wall faces are ignored on input. */
static void load(grid* G, const float* hz, const float* e, const float* u,
                 const float* v) {
  const int64_t nx = G->nx, ny = G->ny;
  int64_t j, k;
  for (j = 1; j <= ny; j++)
    for (k = 1; k <= nx; k++) {
      size_t i = (size_t)(j - 1) * (size_t)nx + (size_t)(k - 1);
      AT(G->H0, j, k) = hz[i];
      AT(G->E, j, k) = e[i];
      AT(G->U, j, k) = (u && k < nx) ? u[i] : 0.0f;
      AT(G->V, j, k) = (v && j < ny) ? v[i] : 0.0f;
    }
}

int sw2d_ref_run(const sw2d_ref_params* p, int64_t nx, int64_t ny,
                 const float* hzero, float* eta, float* u, float* v,
                 int64_t nsteps, double* hist) {
  grid G;
  coeffs c;
  int64_t n, j, k;
  if (bad(p, nx, ny) || !hzero || !eta || !u || !v || nsteps < 0) return -1;
  if (grid_alloc(&G, nx, ny)) return -1;
  load(&G, hzero, eta, u, v);
  c = make_coeffs(p);
  for (n = 0; n < nsteps; n++) {
    step(&G, &c);
    if (hist) reduce(&G, p, hist + (size_t)n * SW2D_REF_NRED);
  }
  for (j = 1; j <= ny; j++)
    for (k = 1; k <= nx; k++) {
      size_t i = (size_t)(j - 1) * (size_t)nx + (size_t)(k - 1);
      eta[i] = AT(G.E, j, k);
      u[i] = (k < nx) ? AT(G.U, j, k) : 0.0f;
      v[i] = (j < ny) ? AT(G.V, j, k) : 0.0f;
    }
  grid_free(&G);
  return 0;
}

int sw2d_ref_reduce(const sw2d_ref_params* p, int64_t nx, int64_t ny,
                    const float* hzero, const float* eta, const float* u,
                    const float* v, double* out) {
  grid G;
  if (bad(p, nx, ny) || !hzero || !eta || !u || !v || !out) return -1;
  if (grid_alloc(&G, nx, ny)) return -1;
  load(&G, hzero, eta, u, v);
  reduce(&G, p, out);
  grid_free(&G);
  return 0;
}

int sw2d_ref_wet(const sw2d_ref_params* p, int64_t nx, int64_t ny,
                 const float* hzero, const float* eta, uint8_t* wet) {
  int64_t i, n;
  if (bad(p, nx, ny) || !hzero || !eta || !wet) return -1;
  n = nx * ny;
  for (i = 0; i < n; i++) wet[i] = (uint8_t)!(hzero[i] + eta[i] < p->hmin);
  return 0;
}
