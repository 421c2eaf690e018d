/* include/sor3d.h — C ABI of the B200-native red-black SOR Poisson solver
 * (the paper's second workload).
 *
 * The operation: the UFLES "press" subroutine of arXiv 1711.04471 §6.3,
 * "Solving of Poisson equation using SOR (iterative solver)" (
 * "solves the Poisson equation for the pressure using Successive
 * Over-Relaxation"), run on "a domain size of 300x300x90,
 * with the number of SOR iterations set to 50"; it is
 * "almost 90% of the run time" on the GPU.  The
 * compiler's "4 reduction kernels" are the solver's
 * convergence folds; here the residual fold is fused into the sweep.  The
 * paper prints no equations: the discretisation and every reading are in
 * DESIGN.md §13 (readings S1-S7):
 *
 *   Lap(p) = cx (p[i+1] + p[i-1]) + cy (p[j+1] + p[j-1]) + cz (p[k+1] + p[k-1])
 *            - dd p,  cx = 1/dx^2, cy = 1/dy^2, cz = 1/dz^2, dd = 2 (cx+cy+cz),
 *   one iteration = red cells (i+j+k even, 1-based interior indices), then
 *   black cells: p <- (1 - omega) p + omega (nsum - rhs) / dd,
 *   residual r = rhs - Lap(p), reported as L2 = sqrt(sum r^2) (fp64) and
 *   Linf = max |r|,
 *   zero Dirichlet values on the ghost layer around the nx x ny x nz
 *   interior.  IEEE binary32, the operation order of DESIGN.md §13.
 *
 * Layout of every host-visible array: float32 [nz][ny][nx] row-major (x
 * fastest), interior values only: a[(k * ny + j) * nx + i], 0-based.
 *
 * Ownership: the caller owns the buffers it passes; the library only reads or
 * writes them during the call (it copies).  Pointers may be host (pageable or
 * pinned) or device (CUDA UVA) memory.  The library owns its device memory
 * and, unless the caller passes one, its CUDA stream.  A handle is not
 * thread-safe.
 *
 * Errors: every int-returning call returns SOR3D_OK (0) or a negative status;
 * nothing aborts and no C++ exception crosses this boundary.  CUDA failures
 * are sticky.  sor3d_last_error() holds a one-line description.
 */
#ifndef SOR3D_H
#define SOR3D_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SOR3D_ABI_VERSION 1

typedef struct sor3d sor3d; /* opaque, library-owned */

enum {
  SOR3D_OK = 0,
  SOR3D_EINVAL = -1, /* bad parameter or non-finite input       */
  SOR3D_ENOMEM = -2, /* device allocation failed                */
  SOR3D_ECUDA = -3,  /* CUDA error (sticky)                     */
  SOR3D_ESTATE = -5  /* iterate/residual/get before sor3d_set   */
};

typedef struct {
  int64_t nx, ny, nz;  /* interior cells, 1 .. 2^20 each; paper: 300, 300, 90     */
  float dx, dy, dz;    /* grid spacings, finite and > 0                           */
  float omega;         /* over-relaxation factor, 0 < omega < 2                   */
  int32_t history_len; /* residual ring capacity (records); 0 -> default 1024     */
} sor3d_params;

/* Library ABI version (SOR3D_ABI_VERSION of the built library). */
int sor3d_abi_version(void);

/* Create a handle on the current device.  cuda_stream: a cudaStream_t to
 * enqueue on, or NULL for a library-owned stream.  Allocates two pressure
 * buffers (ping-pong) and rhs, each padded (DESIGN.md §13 "Layout").
 * SOR3D_EINVAL also if a padded array would reach 2^31 elements (about
 * 1.9e9 cells: the kernel uses 32-bit element offsets).  *out = NULL on
 * failure. */
int sor3d_create(const sor3d_params* params, void* cuda_stream, sor3d** out);

/* Upload p (initial guess; NULL = 0) and rhs, [nz][ny][nx] float32.
 * Synchronous.  SOR3D_EINVAL if any value is non-finite.  Resets the
 * iteration counter and the residual history. */
int sor3d_set(sor3d* h, const float* p, const float* rhs);

/* Enqueue n >= 0 red-black SOR iterations; returns before they complete.  No
 * host<->device transfer.  residual_every = 0: no residual; r > 0: the
 * residual (L2, Linf) after every iteration t (1-based within this call) with
 * t % r == 0, and after the last one, is appended to the history ring; each
 * is computed inside the following iteration's sweep (fused: same loads) or,
 * after the last iteration, by one residual-only pass.  SOR3D_EINVAL if
 * n < 0 or residual_every < 0. */
int sor3d_iterate(sor3d* h, int64_t n, int64_t residual_every);

/* Residual of the current state: out[0] = L2, out[1] = Linf.  Synchronizes. */
int sor3d_residual(sor3d* h, double out[2]);

/* The last n residual records, oldest first, as out[2*t] = L2, out[2*t+1] =
 * Linf; n <= min(records since sor3d_set, history_len).  Synchronizes. */
int sor3d_residual_history(sor3d* h, double* out, int64_t n);

/* Number of residual records appended since sor3d_set (-1 if h is NULL). */
int64_t sor3d_history_count(const sor3d* h);

/* Download p, [nz][ny][nx] float32.  Synchronizes. */
int sor3d_get(sor3d* h, float* p);

/* Wait for all enqueued work of this handle. */
int sor3d_sync(sor3d* h);

/* Number of this library's SOR kernel launches enqueued since create (-1 if
 * h is NULL). */
int64_t sor3d_launch_count(const sor3d* h);

/* One-line description of the launch geometry (tile, z-chunk, CTAs). */
const char* sor3d_plan(const sor3d* h);

/* Destroy the handle and free its device memory.  NULL-safe. */
void sor3d_destroy(sor3d* h);

/* Detail of the last failing call on h (empty if none; h may be NULL for the
 * last sor3d_create failure in this thread). */
const char* sor3d_last_error(const sor3d* h);

#ifdef __cplusplus
}
#endif
#endif /* SOR3D_H */
