/* include/sw2d.h — C ABI of the B200-native 2-D shallow water (2DSW) time step.
 *
 * The operation: the time step of the 2DSW model that arXiv 1711.04471's
 * compiler offloads as map kernels: "a time loop which calls two subroutines,
 * a predictor (dyn) and a first-order Shapiro filter (shapiro), before
 * updating the velocity ... transforms this code into three map-style kernels"
 * (§6.2), run "for 10,000 time steps ... spatial resolution
 * of 1 m and a time step of 0.01 s".  The scheme (the cited
 * textbook's C-grid wet/dry scheme) and every reading of the paper are written
 * out in DESIGN.md ("Oracle step", readings R1-R21).
 *
 * The calls are the domain-level form of the paper's host runtime contract
 * (init, buffer-create, write-buffer, read-buffer, run-kernel,
 * finish) with the paper's transfer minimisation (transfers
 * "made only once in the run"): state is uploaded once by sw2d_set_state and
 * sw2d_step(n) performs no host<->device transfer.
 *
 * Grid and layout (all calls):
 *   nx x ny interior cells; x runs along columns k, y along rows j.
 *   Arakawa C-grid: eta, hzero, wet at cell centres; u[j][k] on the face east
 *   of cell (j,k) (k = nx-1 is the east wall), v[j][k] on the face north of
 *   cell (j,k) (j = ny-1 is the north wall).  West/south walls are implicit
 *   zero faces.  Boundary: closed basin (SW2D_BC_CLOSED).
 *   Host-visible arrays are row-major float32 [nrows][nx] views of the rows
 *   [j0, j0+nrows) this handle owns (the whole grid for one GPU or virtual
 *   ranks): a[(j - j0) * nx + k], 0-based.  Wall-face entries of u and v are
 *   ignored on input and are 0 on output.
 *
 * Ownership: the caller owns every buffer it passes and the library only
 * reads/writes it during the call (it copies).  Pointers may be host
 * (pageable or pinned) or device (CUDA UVA) memory.  The library owns its
 * device memory, its NCCL communicator and, unless the caller passes one, its
 * CUDA stream.  A handle is not thread-safe: one handle per (process, device).
 *
 * Errors: every int-returning call returns SW2D_OK (0) or a negative status;
 * nothing aborts and no C++ exception crosses this boundary.  CUDA and NCCL
 * failures are sticky (every later call returns the same status).
 * sw2d_last_error() holds a one-line description of the last failure.
 */
#ifndef SW2D_H
#define SW2D_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SW2D_ABI_VERSION 4

/* Halo depth (rows) of a row slab: the dependency cone of a two-step pass. */
#define SW2D_HALO_ROWS 4

typedef struct sw2d sw2d; /* opaque, library-owned */

enum {
  SW2D_OK = 0,
  SW2D_EINVAL = -1,      /* bad parameter, non-finite input, nrows < 8 per rank */
  SW2D_ENOMEM = -2,      /* device allocation failed                           */
  SW2D_ECUDA = -3,       /* CUDA error (sticky)                                */
  SW2D_ENCCL = -4,       /* NCCL error or NCCL unavailable (sticky)            */
  SW2D_ESTATE = -5,      /* step/reduce/get before set_state                   */
  SW2D_EUNSUPPORTED = -6 /* e.g. bc != SW2D_BC_CLOSED                          */
};

enum { SW2D_BC_CLOSED = 0 };

/* Diagnostics (reading R16; none in the paper — SPEC.md:406 "0 fold
 * kernels" — the north_star's "global sums and maxima"). */
enum {
  SW2D_RED_VOLUME = 0,    /* dx*dy*sum(hzero + eta) over interior cells, fp64     */
  SW2D_RED_SUM_ETA = 1,   /* sum(eta), fp64                                        */
  SW2D_RED_MAX_ETA = 2,   /* max eta (exact fp32 value)                            */
  SW2D_RED_MIN_ETA = 3,   /* min eta                                               */
  SW2D_RED_MAX_ABS_U = 4, /* max |u| over faces                                    */
  SW2D_RED_MAX_ABS_V = 5, /* max |v|                                               */
  SW2D_RED_WET_COUNT = 6, /* number of wet cells (wet = !(hzero+eta < hmin))       */
  SW2D_RED_N = 7
};

/* Step-kernel variants (sw2d_params.variant). */
enum {
  SW2D_VARIANT_FUSED = 0, /* one fused pass per step: 28 B/cell-step   */
  SW2D_VARIANT_PAPER = 1  /* the paper's shape: three map kernels per step, h and
                             wet stored: 75 B/cell-step; one GPU,
                             no virtual or real ranks; for comparison            */
};

typedef struct {
  int64_t nx, ny;      /* global interior cells, >= 1 each                        */
  float dx, dy, dt;    /* > 0, finite (m, m, s); paper: 1 m, 1 m, 0.01 s          */
  float g;             /* >= 0, finite (g = 0: Shapiro filter only, used by tests) */
  float eps;           /* Shapiro coefficient, 0 <= eps <= 1                      */
  float hmin;          /* wet threshold (m) >= 0: wet iff !(hzero+eta < hmin)     */
  int32_t bc;          /* SW2D_BC_CLOSED                                          */
  uint32_t reduce_every_step; /* bitmask of (1u << SW2D_RED_*) computed inside
                                 every step (fused epilogue) into a history ring */
  int32_t variant;     /* SW2D_VARIANT_*                                          */
  int32_t history_len; /* ring capacity in steps for per-step reductions; 0 ->
                          default 1024                                            */
} sw2d_params;

/* Halo exchange between row slabs (sw2d_dist.halo_mode). */
enum {
  SW2D_HALO_NCCL = 0, /* grouped ncclSend/ncclRecv of the 2 boundary rows on a comm
                         stream, overlapped with the interior launch (default)    */
  SW2D_HALO_P2P = 1   /* fused: the boundary launch of each step stores its rows
                         straight into the neighbours' halo rows (peer memory over
                         NVLink via CUDA IPC; another slab's buffers for virtual
                         ranks) and signals them with stream memory operations.
                         Per-step diagnostics are exchanged the same way: every
                         rank stores its partial record into a slot of every
                         peer and each rank folds the slots in rank order
                         (deterministic, bitwise identical on every rank; no
                         NCCL on the data path)                                  */
};

/* How the ranks of a real multi-rank run find each other (sw2d_dist.bootstrap). */
enum {
  SW2D_BOOT_NCCL = 0,    /* an NCCL communicator from nccl_id (required by
                            SW2D_HALO_NCCL; with SW2D_HALO_P2P it only carries the
                            one-time all-gather of the peer blobs at create)      */
  SW2D_BOOT_EXTERNAL = 1 /* no NCCL at all (SW2D_HALO_P2P only): after create the
                            caller all-gathers every rank's sw2d_p2p_export blob
                            (e.g. over gloo) and passes them to sw2d_p2p_import
                            before sw2d_set_state.  Ranks may share one GPU
                            (CUDA IPC within a device) or sit on peer GPUs      */
};

typedef struct {
  int32_t rank, nranks;  /* row slabs along y (balanced); nrows >= 8 per rank     */
  int32_t device;        /* CUDA ordinal for this rank (-1: current device)       */
  int32_t virtual_ranks; /* 1: run all nranks slabs in this one handle on one
                            device, halos copied device-to-device (no NCCL); the
                            handle then owns the whole grid (test mode)          */
  int32_t halo_mode;     /* SW2D_HALO_*                                           */
  unsigned char nccl_id[128]; /* ncclUniqueId from rank 0 (sw2d_nccl_unique_id),
                                 broadcast by the caller (e.g. torch.distributed);
                                 unused with SW2D_BOOT_EXTERNAL                   */
  int32_t bootstrap;     /* SW2D_BOOT_* (real ranks only)                         */
} sw2d_dist;

/* Library ABI version (SW2D_ABI_VERSION of the built library). */
int sw2d_abi_version(void);

/* Pure host: rows [*j0, *j0 + *nrows) (0-based) of rank `rank` among `nranks`
 * balanced row slabs of a grid with ny rows.  SW2D_EINVAL if nranks < 1, rank
 * out of range, or a slab would have fewer than 2 * SW2D_HALO_ROWS = 8 rows
 * (nranks > 1). */
int sw2d_partition(int64_t ny, int32_t nranks, int32_t rank, int64_t* j0,
                   int64_t* nrows);

/* Pure host: the halo exchange of rank `rank` among `nranks` row slabs, done
 * before every pass of one or two steps (the dependency cone of two steps is
 * SW2D_HALO_ROWS = 4 rows: DESIGN.md "Multi-GPU").  A slab's fields are
 * (nrows + 8)-row arrays: storage rows 0..3 are the south halo, 4 .. nrows+3
 * the owned rows, nrows+4 .. nrows+7 the north halo.  Each message is
 * SW2D_HALO_ROWS consecutive storage rows of eta, u and v (of hzero once, in
 * sw2d_set_state).  out[0] = first row sent to the south neighbour (rank-1),
 * out[1] = first row received from it, out[2] = first row sent to the north
 * neighbour (rank+1), out[3] = first row received from it; -1 where there is
 * no neighbour.  Returns the number of neighbours (0..2) or SW2D_EINVAL (as
 * sw2d_partition).  The library performs the exchange; this is its plan. */
int sw2d_halo_plan(int64_t ny, int32_t nranks, int32_t rank, int64_t out[4]);

/* Pure host: writes a fresh ncclUniqueId (128 bytes) for sw2d_dist.nccl_id.
 * SW2D_ENCCL if NCCL cannot be loaded. */
int sw2d_nccl_unique_id(unsigned char out[128]);

/* Bytes of one rank's peer blob (sw2d_p2p_export / sw2d_p2p_import). */
#define SW2D_P2P_BLOB_BYTES 1024

/* Create a handle.  dist == NULL: one GPU (the current device), whole grid.
 * cuda_stream: a cudaStream_t to enqueue on (e.g. torch's current stream), or
 * NULL for a library-owned stream.  Allocates 7 device arrays (hzero and
 * double-buffered eta, u, v) of (nrows + 8) x pitch floats.  *out = NULL on
 * failure. */
int sw2d_create(const sw2d_params* params, const sw2d_dist* dist,
                void* cuda_stream, sw2d** out);

/* P2P mode across real ranks (SW2D_HALO_P2P; SURVEY.md §8(e) "Fused P2P
 * alternative"): write this rank's peer blob — its grid geometry and the CUDA
 * IPC handles of its state buffers (eta, u, v double-buffered, hzero) and of
 * its sync buffer (halo flags, the record-exchange flags and slots) — into
 * out[0 .. SW2D_P2P_BLOB_BYTES).  The blob is plain bytes: the caller moves it
 * to every rank (any transport).  SW2D_EINVAL if the handle is not a real
 * rank in P2P mode. */
int sw2d_p2p_export(sw2d* h, void* out, size_t cap);

/* Map the peers: `blobs` holds nranks blobs of SW2D_P2P_BLOB_BYTES each, in
 * rank order (rank r's own blob at r, as exported).  Opens the row
 * neighbours' state buffers and every peer's sync buffer (CUDA IPC; peer GPUs
 * over NVLink with lazy peer access, or the same GPU).  Checks that every
 * blob describes the same grid and partition (SW2D_EINVAL otherwise).  Call
 * once, after create and before sw2d_set_state, on every rank (with
 * SW2D_BOOT_NCCL, create has already done it). */
int sw2d_p2p_import(sw2d* h, const void* blobs, size_t nbytes);

/* Rows [*j0, *j0 + *nrows) (0-based, global) whose state this handle holds. */
int sw2d_local_rows(const sw2d* h, int64_t* j0, int64_t* nrows);

/* Shape of the host-visible [nrows][nx] arrays of this handle (the rows of
 * sw2d_local_rows, the global nx): what set_state reads and get_state writes
 * per field. */
int sw2d_local_shape(const sw2d* h, int64_t* nrows, int64_t* nx);

/* Upload the state (the paper's once-per-run write-buffer): hzero, eta, u, v
 * as [nrows][nx] float32 (see layout above).  u and v may be NULL (= 0).
 * Synchronous.  SW2D_EINVAL if any interior value is non-finite.  Resets the
 * step counter and the reduction history.  With nranks > 1 every rank must
 * call it (it exchanges the static hzero halo once). */
int sw2d_set_state(sw2d* h, const float* hzero, const float* eta,
                   const float* u, const float* v);

/* Enqueue nsteps >= 0 time steps on the handle's stream; returns before they
 * complete.  No host<->device transfer.  Steps run two per launch where the
 * kernels allow it, and long calls in one process replay CUDA graphs.  With
 * nranks > 1 it exchanges the SW2D_HALO_ROWS-row halos before every pass of
 * one or two steps (NCCL send/recv, or fused P2P stores) and, if
 * reduce_every_step != 0, combines the per-step diagnostics of all ranks
 * (NCCL allreduce, or the P2P slot exchange) into every rank's history.
 * Every rank must make the same sequence of sw2d_set_state / sw2d_step /
 * sw2d_reduce calls (collective). */
int sw2d_step(sw2d* h, int64_t nsteps);

/* Periodic output (the paper's once-per-run / per-iteration transfer
 * scheduling): run nsteps steps and
 * deliver eta after every `every` steps: out_eta[k] ([nrows][nx] float32, the
 * rows this handle holds) = eta after (k+1)*every steps, k < nsnap =
 * nsteps / every.  Each snapshot is packed on the device into one of two
 * staging buffers and copied to the host on a copy stream while the following
 * steps run (use pinned host memory for the overlap).  Synchronizes before
 * returning.  SW2D_EINVAL if every < 1 or nsnap != nsteps / every. */
int sw2d_run_snapshots(sw2d* h, int64_t nsteps, int64_t every, float* out_eta,
                       int64_t nsnap);

/* The global value of diagnostic `op` (SW2D_RED_*) of the current state, on
 * every rank.  Synchronizes. */
int sw2d_reduce(sw2d* h, int op, double* out);

/* The per-step values of diagnostic `op` for the last n steps (oldest first),
 * n <= min(steps taken since set_state, history_len); op must be in
 * reduce_every_step.  Synchronizes. */
int sw2d_reduce_history(sw2d* h, int op, double* out, int64_t n);

/* Download the state rows this handle holds: eta, u, v [nrows][nx] float32 and
 * wet [nrows][nx] uint8 (0/1).  Any pointer may be NULL.  Synchronizes. */
int sw2d_get_state(sw2d* h, float* eta, float* u, float* v, uint8_t* wet);

/* Wait for all enqueued work of this handle. */
int sw2d_sync(sw2d* h);

/* Number of this library's kernel launches enqueued since create (all kinds);
 * -1 if h is NULL. */
int64_t sw2d_launch_count(const sw2d* h);

/* One-line description of the step plan this handle runs (kernel family,
 * model steps per launch, launches per pass, strips, CTAs per SM, halo mode);
 * owned by the handle, valid until sw2d_destroy.  "" if h is NULL. */
const char* sw2d_plan(const sw2d* h);

/* Destroy the handle and free its device memory / communicator.  NULL-safe. */
void sw2d_destroy(sw2d* h);

/* Static description of a status code. */
const char* sw2d_strerror(int code);

/* Detail of the last failing call on h (empty string if none; h may be NULL
 * for the last sw2d_create failure in this thread). */
const char* sw2d_last_error(const sw2d* h);

#ifdef __cplusplus
}
#endif
#endif /* SW2D_H */
