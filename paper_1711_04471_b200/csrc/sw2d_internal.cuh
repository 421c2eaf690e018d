// paper_1711_04471_b200/csrc/sw2d_internal.cuh — internal types shared by the
// CUDA kernels (sw2d_kernels.cu) and the host runtime (sw2d_host.cu).
//
// Device layout: every field of a slab is a
// row-major float32 array of (nrows + 8) rows x `pitch` floats.  Storage row
// r holds global 1-based row j = jbase + r (jbase = first owned row - 4, so
// four halo rows sit on each side: the dependency cone of a two-step pass).  Storage column c holds 1-based interior
// column k = c - kColOff (k = 1 at c = 8; the west wall halo column k = 0 is
// c = 7).  Warp strip s reads storage columns [120 s + 4, 120 s + 132) and
// writes [120 s + 8, 120 s + 128): 15 whole 32-byte sectors, so no sector is
// written by two warps.  pitch is a multiple of 32 floats (128 B).
#pragma once
#include <cstdint>
#include <cstdio>

namespace sw2d_dev {

constexpr int kColOff = 7;           // storage column of 1-based column k is k + 7
constexpr int kStripBase = kColOff - 3;  // storage column where strip 0's window starts
constexpr int kHaloRows = 4;         // halo rows per side: the cone of a two-step pass
constexpr int kWarpsPerBlock = 4;      // grid-stride helper kernels
constexpr int kThreads = 32 * kWarpsPerBlock;
constexpr int kOutLanes = 30;        // lanes 1..30 produce output; 0 and 31 are halo lanes
constexpr int kColsPerStrip = 4 * kOutLanes;   // 120 output columns per warp strip

// Model coefficients, computed once on the host in double and rounded once
// (reading R12).
struct Coef {
  float cgx, cgy, cx, cy, q, hmin;
  float nz;  // -0.0f: the addend of the packed products (a kernel parameter, so
             // ptxas cannot fold fma(a, b, -0) into a multiply and contract it)
};

// One slab's fields: state n (read) and state n+1 (written).
struct SlabView {
  const float* E;
  const float* U;
  const float* V;
  const float* H0;
  float* En;
  float* Un;
  float* Vn;
  long long pitch;   // floats per storage row
  long long jbase;   // global 1-based row of storage row 0
  long long nelem;   // floats per field allocation (bounds checks in debug builds)
};

// Debug builds (python -m paper_1711_04471_b200._build --debug): every global
// store and TMA window of the step kernels is bounds-checked on the device.
#ifdef SW2D_DEBUG_BOUNDS
#define SW2D_CHECK(cond)                                                     \
  do {                                                                       \
    if (!(cond)) {                                                           \
      printf("sw2d bounds check failed: %s (%s:%d) block %d thread %d\n",    \
             #cond, __FILE__, __LINE__, (int)blockIdx.x, (int)threadIdx.x);   \
      __trap();                                                              \
    }                                                                        \
  } while (0)
#else
#define SW2D_CHECK(cond) \
  do {                   \
  } while (0)
#endif

// Per-step diagnostics record (7 doubles, see SW2D_RED_*): the sum part
// [0..2] and the max part [3..6] are allreduced separately across ranks.
enum { kRecVol = 0, kRecSumEta = 1, kRecWet = 2, kRecMaxEta = 3,
       kRecNegMinEta = 4, kRecMaxU = 5, kRecMaxV = 6, kRecN = 7 };

// Per-CTA partial of the diagnostics.
struct RedPartial {
  double sum_eta;
  double wet;
  float max_eta, neg_min_eta, max_u, max_v;
};

struct RedArgs {
  RedPartial* partials;      // one slot per CTA of the step (all launches)
  int part_base;             // first slot of this launch
  unsigned int* counter;     // CTAs done this step (reset by the last CTA)
  int expected;              // CTAs writing partials this step (all launches)
  double* rec;               // the step's 7-double record (written by last CTA)
  const double* h0sum;       // sum of hzero over the cells this handle owns
  double dxdy;
};

// Fused halo (P2P mode): output rows [lo, hi] (global, 1-based) are also
// stored into a neighbour slab's state n+1 fields — another slab on this GPU
// (virtual ranks) or a peer GPU's buffers mapped over NVLink (CUDA IPC).
struct Remote {
  float* En;
  float* Un;
  float* Vn;
  long long jbase;   // the neighbour slab's global 1-based row of storage row 0
  long long nelem;   // floats per field of the neighbour slab (debug bounds checks)
  int lo, hi;        // rows to mirror; lo > hi: none
};

struct StepArgs {
  SlabView s;
  Remote rem[2];             // used by the boundary launches in P2P halo mode
  int nx;
  long long ny;
  long long row_lo, row_hi;  // global 1-based output rows of this launch (inclusive)
  int rows_per_seg;          // output rows per warp segment
  int nstrips;               // warp strips across the columns
  int nsegs;                 // warp segments down the rows
  int sk_ctas;               // two-step kernel: 0 = group x segment grid; > 0 = this many
                             // CTAs sharing the strip-rows evenly (one per SM)
  Coef c;
  RedArgs red;
  RedArgs red2;              // two-step launches: the second step's record
};

// Step-kernel launchers (sw2d_kernels.cu).  `red_level`: 0 none, 1 sums
// (VOLUME, SUM_ETA), 2 all diagnostics.  `kind`: 1 = CTA of kCtaStrips
// compute warps + a producer warp sharing one TMA row ring (default); 2 =
// small grids: 2 columns per lane, plain loads, 4 independent warps per CTA.
int step_strips_per_cta(int kind);
int step_strip_cols(int kind);   // output columns per warp strip (120, or 60 for kind 2)
int step_grid(int kind, int nstrips, int nsegs);   // CTAs of one step launch
void launch_step(const StepArgs& a, int red_level, int kind, void* stream,
                 bool remote = false);
int step_occupancy_blocks_per_sm(int red_level, int kind);
// Two steps per launch (kind 1 layout, one slab): state n -> n+2.
void launch_step2(const StepArgs& a, int red_level, void* stream, bool remote = false);
// its three diagnostics levels, each built in a translation unit of its own
// (sw2d_cta2_r0.cu, _r1.cu, _r2.cu)
void launch_step2_r0(const StepArgs& a, void* stream, bool remote);
void launch_step2_r1(const StepArgs& a, void* stream, bool remote);
void launch_step2_r2(const StepArgs& a, void* stream, bool remote);
int step2_strips_per_cta();
void launch_step2_small(const StepArgs& a, int red_level, void* stream,
                        bool defer = false);  // kind 2, two steps
// fold `nsteps` steps' deferred partials (`blocks` per step) into history slots
// (*dstep + s) % len
void launch_fold_steps(const RedPartial* partials, int blocks, int nsteps, double* hist, int len,
                       const unsigned long long* dstep, const double* h0sum, double dxdy,
                       void* stream);
int step2_small_occupancy_blocks_per_sm(int red_level);
int step2_small_strip_cols();  // 56

// set_state helper: checks finiteness of the interior, zeroes the wall faces
// of U (k = nx) and V (global j = ny), and sums hzero in fp64 into *h0sum.
struct IngestArgs {
  float* E;
  float* U;
  float* V;
  const float* H0;
  long long pitch;
  long long jbase;           // global 1-based row of storage row 0
  long long nrows;           // owned rows (storage rows 2 .. nrows+1)
  int nx;
  long long ny;
  int* bad;                  // set to 1 if any value is non-finite
  RedArgs red;               // partials/counter/expected; result into *red.rec (1 double)
};
int ingest_blocks(const IngestArgs& a);
void launch_ingest(const IngestArgs& a, void* stream);

// Diagnostics of the current state (sw2d_reduce): same record as the fused
// epilogue.  One launch per slab; all slabs of a handle share the counter.
struct ReduceArgs {
  const float* E;
  const float* U;
  const float* V;
  const float* H0;
  long long pitch;
  long long nrows;
  int nx;
  float hmin;
  RedArgs red;
};
int reduce_blocks(const ReduceArgs& a);
void launch_reduce(const ReduceArgs& a, void* stream);

// The paper-shaped unfused step (sw2d_paper_kernels.cu): three map kernels
// per step, h and wet stored (SW2D_VARIANT_PAPER).
struct PaperArgs {
  const float* E;            // state n: eta, u, v (read by K1/K2)
  const float* U;
  const float* V;
  const float* H0;
  float* un;                 // scratch: K1 -> K2, K3
  float* vn;
  float* etan;               // scratch: K2 -> K3
  float* h;                  // stored depth (K3 writes, K2 reads next step)
  const unsigned char* wet_in;   // start-of-step wet flags
  unsigned char* wet_out;        // end-of-step wet flags
  float* Eo;                 // state n+1 (in place: K3 writes E, U, V)
  float* Uo;
  float* Vo;
  long long pitch;           // elements per storage row (floats and flags)
  long long jbase;
  long long nrows;
  int nx;
  long long ny;
  Coef c;
};
void launch_paper_step(const PaperArgs& a, void* stream);   // 3 launches
void launch_paper_init(const PaperArgs& a, void* stream);   // h, wet_out from H0 + E


// Persistent cooperative kernel for small grids (sw2d_persist.cu): one launch
// advances a whole grid `nsteps` steps; CTA t owns tile t (ntx x nty tiles of
// (64 - 4K) x th cells), K steps per shared-memory block, neighbour tiles
// synchronised through per-tile step counters.
struct PersistArgs {
  float* E[2];
  float* U[2];
  float* V[2];
  const float* H0;
  long long pitch;
  long long jbase;           // global 1-based row of storage row 0
  int nx, ny;
  int shape;                 // CTA shape (persist_shape_*)
  int th;                    // tile rows (persist_tile_rows)
  int ntx, nty;              // tiles across / down
  int cur;                   // buffer holding the state at the first step
  int nsteps;
  unsigned* flags;           // per tile: steps published (monotone across launches)
  unsigned flag_base;        // the value every flag reached before this launch (and
                             // the tag base of the ring words)
  unsigned long long* ring;  // tagged ring words [2][3][ny][nx] (tag << 32 | value
                             // bits) instead of counters; nullptr: counters
  long long ring_plane;      // nx * ny
  Coef c;
  RedPartial* part;          // [nsteps][ntiles] per-step CTA partials (RED >= 1)
};
// CTA shapes (0 .. persist_shapes()-1): warps per CTA x shared rows per thread
int persist_shapes();
int persist_shape_rows(int shape);       // shared-tile rows
int persist_shape_warps(int shape);
int persist_tile_cols(int K);
int persist_tile_rows(int K, int shape);
size_t persist_flag_words(int ntiles);   // flag array length (one 128-byte line per tile)
size_t persist_ring_words(long long nx, long long ny);   // tagged ring words
int persist_capacity(int K, int red_level, int shape);   // co-resident CTAs
int launch_persist(const PersistArgs& a, int K, int red_level, void* stream);  // 0 or cudaError

// wet mask of the current state into a dense uint8 [nrows][nx] buffer.
void launch_wet(const float* E, const float* H0, long long pitch,
                long long nrows, int nx, float hmin, unsigned char* out,
                void* stream);

}  // namespace sw2d_dev
