/* oracle/sw2d_ref.h — TEST INFRASTRUCTURE ONLY.
 *
 * Declarations for the plain, single-threaded C11 oracle of the 2-D shallow
 * water (2DSW) time step of arXiv 1711.04471 §6.2.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load it.  It shares no header, helper or constant
 * generator with the CUDA product path (paper_1711_04471_b200/, include/).
 *
 * Arrays are host, row-major, unpadded: a[j*nx + k], j = 0..ny-1 (y, rows),
 * k = 0..nx-1 (x, columns).  u[j][k] is the face east of cell (j,k) (k = nx-1
 * is the east wall), v[j][k] the face north of cell (j,k) (j = ny-1 is the
 * north wall).  West/south walls are implicit zero faces.  All state is IEEE
 * binary32 (reading #11 in DESIGN.md).
 */
#ifndef SW2D_REF_H
#define SW2D_REF_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* reduction slots written by sw2d_ref_reduce / the per-step history */
enum {
  SW2D_REF_VOLUME = 0,     /* dx*dy*sum(H0 + eta) over interior cells (fp64)   */
  SW2D_REF_SUM_ETA = 1,    /* sum(eta) (fp64, Neumaier)                         */
  SW2D_REF_MAX_ETA = 2,    /* max eta over interior cells (exact fp32)          */
  SW2D_REF_MIN_ETA = 3,    /* min eta                                           */
  SW2D_REF_MAX_ABS_U = 4,  /* max |u| over faces                                */
  SW2D_REF_MAX_ABS_V = 5,  /* max |v|                                           */
  SW2D_REF_WET_COUNT = 6,  /* number of wet cells, wet = !(H0+eta < hmin)       */
  SW2D_REF_NRED = 7
};

typedef struct {
  float dx, dy, dt, g, eps, hmin;
} sw2d_ref_params;

/* Advance (eta, u, v) in place by nsteps.  hist (nullable) receives
 * nsteps * SW2D_REF_NRED doubles: the reductions of the state after each step.
 * Returns 0, or -1 on bad arguments / allocation failure. */
int sw2d_ref_run(const sw2d_ref_params* p, int64_t nx, int64_t ny,
                 const float* hzero, float* eta, float* u, float* v,
                 int64_t nsteps, double* hist);

/* The seven diagnostics of the current state into out[SW2D_REF_NRED]. */
int sw2d_ref_reduce(const sw2d_ref_params* p, int64_t nx, int64_t ny,
                    const float* hzero, const float* eta, const float* u,
                    const float* v, double* out);

/* wet[j*nx+k] = !(hzero+eta < hmin) as 0/1 bytes. */
int sw2d_ref_wet(const sw2d_ref_params* p, int64_t nx, int64_t ny,
                 const float* hzero, const float* eta, uint8_t* wet);

#ifdef __cplusplus
}
#endif
#endif
