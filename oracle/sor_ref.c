/* oracle/sor_ref.c — TEST INFRASTRUCTURE ONLY (the parity oracle of NEXT-4).
 *
 * A plain single-threaded C11 red-black SOR solver for the Poisson equation,
 * the UFLES "press" hot spot of arXiv 1711.04471 §6.3 ("solves the Poisson
 * equation for the pressure using Successive Over-Relaxation",
 * PAPER.md:399-401, 418; "300x300x90, with the number of SOR iterations set
 * to 50"; the compiler's "4 reduction kernels" are the
 * convergence folds).  The paper gives no equations; the
 * readings (S1-S7): 7-point Laplacian on a node grid with
 * spacings dx, dy, dz and zero Dirichlet ghosts, red-black ordering by the
 * parity of i+j+k (1-based interior indices, red = even), over-relaxation
 * factor omega, IEEE binary32 arithmetic in the order written below (built
 * with -ffp-contract=off -fno-fast-math), residual r = rhs - Lap(p) folded as
 * L2 = sqrt(sum r^2) (fp64, Neumaier) and Linf = max |r| (exact fp32).
 *
 * Only tests/, __graft_entry__ and bench.py's reference leg load it; it
 * shares no code with the CUDA path.
 *
 * Arrays: host, [nz][ny][nx] row-major (x fastest), interior values only.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  float dx, dy, dz, omega;
} sor_ref_params;

#define P3(a, k, j, i) \
  (a)[((size_t)(k) * (size_t)(ny + 2) + (size_t)(j)) * (size_t)(nx + 2) + (size_t)(i)]

typedef struct {
  float cx, cy, cz, dd, invd, om, om1;
} sor_coef;

/* coefficients once, in double, one rounding each (reading S4) */
static sor_coef make_coef(const sor_ref_params* p) {
  sor_coef c;
  const double ax = 1.0 / ((double)p->dx * (double)p->dx);
  const double ay = 1.0 / ((double)p->dy * (double)p->dy);
  const double az = 1.0 / ((double)p->dz * (double)p->dz);
  c.cx = (float)ax;
  c.cy = (float)ay;
  c.cz = (float)az;
  c.dd = (float)(2.0 * (ax + ay + az));
  c.invd = (float)(1.0 / (2.0 * (ax + ay + az)));
  c.om = p->omega;
  c.om1 = (float)(1.0 - (double)p->omega);
  return c;
}

/* neighbour sum of the 7-point stencil: (cx*(E+W) + cy*(N+S)) + cz*(U+D) */
static float nsum(const float* p, int64_t nx, int64_t ny, int64_t k, int64_t j, int64_t i,
                  const sor_coef* c) {
  const float sx = c->cx * (P3(p, k, j, i + 1) + P3(p, k, j, i - 1));
  const float sy = c->cy * (P3(p, k, j + 1, i) + P3(p, k, j - 1, i));
  const float sz = c->cz * (P3(p, k + 1, j, i) + P3(p, k - 1, j, i));
  return (sx + sy) + sz;
}

/* one red-black SOR iteration: the red cells (i+j+k even), then the black */
static void sweep(float* p, const float* rhs, int64_t nx, int64_t ny, int64_t nz,
                  const sor_coef* c) {
  for (int colour = 0; colour < 2; ++colour)
    for (int64_t k = 1; k <= nz; ++k)
      for (int64_t j = 1; j <= ny; ++j)
        for (int64_t i = 1; i <= nx; ++i) {
          if (((i + j + k) & 1) != colour) continue;
          const float s = nsum(p, nx, ny, k, j, i, c) - P3(rhs, k, j, i);
          P3(p, k, j, i) = c->om1 * P3(p, k, j, i) + c->om * (s * c->invd);
        }
}

typedef struct { double s, c; } nsum_t;
static void nadd(nsum_t* a, double x) {
  const double t = a->s + x;
  if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x;
  else a->c += (x - t) + a->s;
  a->s = t;
}

/* residual r = rhs - Lap(p), Lap(p) = nsum - dd*p: out[0] = L2, out[1] = Linf */
static void residual(const float* p, const float* rhs, int64_t nx, int64_t ny, int64_t nz,
                     const sor_coef* c, double* out) {
  nsum_t s2 = {0.0, 0.0};
  float mx = 0.0f;
  for (int64_t k = 1; k <= nz; ++k)
    for (int64_t j = 1; j <= ny; ++j)
      for (int64_t i = 1; i <= nx; ++i) {
        const float lap = nsum(p, nx, ny, k, j, i, c) - c->dd * P3(p, k, j, i);
        const float r = P3(rhs, k, j, i) - lap;
        nadd(&s2, (double)r * (double)r);
        if (fabsf(r) > mx) mx = fabsf(r);
      }
  out[0] = sqrt(s2.s + s2.c);
  out[1] = mx;
}

static float* halo_copy(const float* a, int64_t nx, int64_t ny, int64_t nz) {
  float* h = calloc((size_t)(nx + 2) * (size_t)(ny + 2) * (size_t)(nz + 2), sizeof(float));
  if (!h) return NULL;
  for (int64_t k = 1; k <= nz; ++k)
    for (int64_t j = 1; j <= ny; ++j)
      memcpy(&P3(h, k, j, 1), a + ((size_t)(k - 1) * ny + (size_t)(j - 1)) * nx,
             (size_t)nx * sizeof(float));
  return h;
}

static int bad(const sor_ref_params* p, int64_t nx, int64_t ny, int64_t nz) {
  return !p || nx < 1 || ny < 1 || nz < 1 || !(p->dx > 0.0f) || !(p->dy > 0.0f) ||
         !(p->dz > 0.0f) || !(p->omega > 0.0f && p->omega < 2.0f);
}

/* n red-black iterations in place on p; hist (nullable) receives 2 doubles
 * (L2, Linf) of the residual after each iteration. */
int sor_ref_run(const sor_ref_params* prm, int64_t nx, int64_t ny, int64_t nz, float* p,
                const float* rhs, int64_t n, double* hist) {
  if (bad(prm, nx, ny, nz) || !p || !rhs || n < 0) return -1;
  const sor_coef c = make_coef(prm);
  float* hp = halo_copy(p, nx, ny, nz);
  float* hr = halo_copy(rhs, nx, ny, nz);
  if (!hp || !hr) {
    free(hp);
    free(hr);
    return -1;
  }
  for (int64_t it = 0; it < n; ++it) {
    sweep(hp, hr, nx, ny, nz, &c);
    if (hist) residual(hp, hr, nx, ny, nz, &c, hist + 2 * it);
  }
  for (int64_t k = 1; k <= nz; ++k)
    for (int64_t j = 1; j <= ny; ++j)
      memcpy(p + ((size_t)(k - 1) * ny + (size_t)(j - 1)) * nx, &P3(hp, k, j, 1),
             (size_t)nx * sizeof(float));
  free(hp);
  free(hr);
  return 0;
}

/* residual of a state: out[0] = L2, out[1] = Linf */
int sor_ref_residual(const sor_ref_params* prm, int64_t nx, int64_t ny, int64_t nz,
                     const float* p, const float* rhs, double* out) {
  if (bad(prm, nx, ny, nz) || !p || !rhs || !out) return -1;
  const sor_coef c = make_coef(prm);
  float* hp = halo_copy(p, nx, ny, nz);
  float* hr = halo_copy(rhs, nx, ny, nz);
  if (!hp || !hr) {
    free(hp);
    free(hr);
    return -1;
  }
  residual(hp, hr, nx, ny, nz, &c, out);
  free(hp);
  free(hr);
  return 0;
}
