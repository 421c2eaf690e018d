// paper_1711_04471_b200/csrc/sw2d_host.cu — host runtime behind include/sw2d.h.
//
// Owns the device state of one handle (one GPU, or all virtual ranks on one
// GPU), plans the step-kernel launches, runs the time loop without host
// transfers (the paper's once-per-run transfer rule), moves
// the 2-row halos between row slabs (NCCL send/recv over NVLink between
// ranks, device copies between virtual ranks) and folds the diagnostics.
// See DESIGN.md "Host runtime" and "Multi-GPU".
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "sw2d.h"
#include <nvtx3/nvToolsExt.h>
#include "sw2d_internal.cuh"
#include "sw2d_nccl.cuh"

using namespace sw2d_dev;

namespace {

thread_local std::string t_create_err;

std::mutex g_persist_mu;                  // orders persistent launches per device
cudaEvent_t g_persist_last[64] = {};

constexpr long long kSmallMaxCells = 1LL << 21;   // small-grid kernel up to ~1448^2
constexpr int kMinRowsPerSeg = 4;
constexpr int kGraphPasses = 32;  // passes per captured CUDA graph (even)

bool graphs_enabled() {
  const char* e = std::getenv("SW2D_GRAPHS");
  return !(e && std::atoi(e) == 0);
}   // small grids: more, shorter segments (latency-bound)
constexpr int kDefaultHistory = 1024;

struct Slab {
  int64_t j0 = 0, nrows = 0;  // 0-based global first owned row, owned rows
  float* Hs = nullptr;                     // paper variant: stored depth h
  unsigned char* W[2] = {nullptr, nullptr};  // paper variant: wet flags
  float* H0 = nullptr;
  float* E[2] = {nullptr, nullptr};
  float* U[2] = {nullptr, nullptr};
  float* V[2] = {nullptr, nullptr};
};

// One step-kernel launch over a band of rows of one slab.
struct Launch {
  int slab;
  long long row_lo, row_hi;  // global 1-based rows, inclusive
  int rows_per_seg, nsegs, blocks, part_base;
  int phase;                 // 0: needs no halo of this step; 1: after the halo exchange
  int sk = 0;                // two-step kernel: CTAs sharing the strip-rows evenly (0: off)
};

}  // namespace

struct sw2d {
  sw2d_params p{};
  Coef coef{};
  int rank = 0, nranks = 1;
  bool virt = false, multi = false;  // multi: real ranks (NCCL or P2P transport)
  int bootstrap = SW2D_BOOT_NCCL;    // real ranks: SW2D_BOOT_*
  int device = 0;
  int64_t pitch = 0;
  int nstrips = 0;
  int red_level = 0;
  int nstrips2 = 0;  // kind 2, two steps per launch: 56-column strips
  int64_t fault_skip_halo = -1;  // SW2D_FAULT_SKIP_HALO (tests only)
  int kind = 1;  // step kernel kind (sw2d_internal.cuh); SW2D_STEP_KERNEL overrides
  // persistent cooperative kernel (small grids): K steps per shared-memory
  // block, pntx x pnty tiles of pth rows, one CTA each; pk = 0: off
  int pk = 0, pshape = 0, pth = 0, pntx = 0, pnty = 0;
  bool ptag = false;   // tagged ring words instead of per-tile counters
  unsigned* pflags = nullptr;   // per-tile step counters
  unsigned long long* pring = nullptr;   // tagged ring words (plans with one CTA per SM)
  unsigned pbase = 0;           // their value before the next launch
  RedPartial* ppart = nullptr;  // per-step CTA partials of one launch chunk
  std::vector<Slab> slabs;
  std::vector<Launch> launches;
  int step_blocks = 0;
  std::vector<Launch> launches2;  // two steps per launch (kind 1): empty if unavailable
  int step_blocks2 = 0;
  int cur = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t comm = nullptr;
  cudaEvent_t ev_ready = nullptr, ev_halo = nullptr;
  RedPartial* partials = nullptr;
  int partials_cap = 0;
  unsigned int* counter = nullptr;
  // CUDA graphs with per-step diagnostics: a captured pass writes its records
  // to grec[step within the graph]; the graph ends with ring_scatter, which
  // moves them to the history ring at the device step counter *dstep.
  double* grec = nullptr;
  unsigned long long* dstep = nullptr;
  bool capturing = false;
  int cap_step = 0;
  RedPartial* gpart = nullptr;  // deferred partials of a captured graph's steps (small grids)
  double* hist = nullptr;
  int hist_len = 0;
  double* rec = nullptr;    // scratch record (ingest, sw2d_reduce)
  double* h0sum = nullptr;  // sum of hzero over the cells this handle owns
  double* zero = nullptr;   // a device 0.0
  int* bad = nullptr;
  int* bad_host = nullptr;   // mapped pinned host word: set_state's verdict without a DMA
  unsigned char* wetbuf = nullptr;
  size_t wetbuf_bytes = 0;
  float* stage = nullptr;   // dense [field][rows][nx] staging of host transfers (1D DMA)
  size_t stage_floats = 0;
  float* snap[2] = {nullptr, nullptr};   // periodic-output staging buffers
  size_t snap_bytes = 0;
  cudaStream_t copy = nullptr;
  cudaEvent_t ev_snap[2] = {nullptr, nullptr}, ev_copied[2] = {nullptr, nullptr};
  int64_t steps = 0;
  int wcur = 0;  // paper variant: current wet buffer
  bool state_set = false;
  // records of real ranks: each pass's kernels write this rank's partial
  // record of exchange sequence number q to its own slot xslot[q % kXRing]
  // [rank] of the sync buffer; the comm stream combines the ranks' slots into
  // the destination (history slot or scratch): NCCL allreduce (out of place),
  // or in P2P mode the slot exchange (every rank stores its record into every
  // peer's slot, each folds in rank order).  ev_x[q % kXRing] is recorded on
  // the comm stream once record q is combined; the compute stream waits on it
  // before a kernel reuses the slot.
  struct PendingRec {
    uint64_t seq;
    double* dst;
  };
  std::vector<PendingRec> pending;  // records awaiting the NCCL allreduce
  uint64_t xseq = 0;                // records exchanged so far (never reset)
  uint32_t hseq = 0;                // P2P halo signals sent to each neighbour (never reset)
  unsigned char* sync = nullptr;    // flags + record slots (IPC-exported in P2P mode)
  size_t sync_bytes = 0;
  std::vector<unsigned char*> psync;  // every peer's sync buffer, IPC-mapped (P2P)
  bool p2p_ready = false;           // P2P peers mapped (sw2d_p2p_import)
  cudaEvent_t ev_x[64] = {};
  // CUDA graphs of kGraphPasses passes (one slab, no per-step diagnostics),
  // one per starting buffer parity; replayed for long sw2d_step calls
  cudaGraphExec_t graph[2] = {nullptr, nullptr};
  int graph_spl = 0;
  std::string plan_text;  // sw2d_plan()
  int sticky = 0;
  std::string err;
  ncclComm_t comm_nccl = nullptr;
  int64_t nlaunch = 0;
  // P2P halo mode
  int halo_mode = SW2D_HALO_NCCL;
  struct Peer {
    bool present = false;
    float* E[2] = {nullptr, nullptr};
    float* U[2] = {nullptr, nullptr};
    float* V[2] = {nullptr, nullptr};
    float* H0 = nullptr;
    long long jbase = 0;
    long long nelem = 0;
    long long nrows = 0;
  } nbr[2];                       // [0]: south (rank-1), [1]: north (rank+1); IPC-mapped
};

namespace {

// --- real ranks: the sync buffer --------------------------------------------
// One device allocation per rank (IPC-exported in P2P mode), zeroed at create:
//   bytes [0, 8)          halo flags: [0] written by the south neighbour, [1]
//                         by the north one (P2P: halo signals received so far)
//   bytes [64, 64+4P)     xflag[q]: records rank q has stored into this rank's slots
//   bytes [.., +4P)       xack[q]:  records rank q has folded (its slots reusable)
//   from sync_slots(P)    double slots[kXRing][P][kRecN]: record q of rank r at
//                         [q % kXRing][r]
// Flag values count events since create and are never reset (no epoch race
// between a neighbour's last signal of one run and the next sw2d_set_state).
constexpr int kXRing = 64;
constexpr int kMaxRanks = 128;
static_assert(kXRing == sizeof(((sw2d*)nullptr)->ev_x) / sizeof(cudaEvent_t), "ev_x size");
size_t sync_xflag() { return 64; }
size_t sync_xack(int P) { return 64 + 4 * (size_t)P; }
size_t sync_slots(int P) { return (64 + 8 * (size_t)P + 255) / 256 * 256; }
size_t sync_size(int P) { return sync_slots(P) + sizeof(double) * kRecN * kXRing * (size_t)P; }
unsigned long long flag_addr(unsigned char* sync, size_t off, int i) {
  return (unsigned long long)(sync + off + 4 * (size_t)i);
}
double* xslot(unsigned char* sync, int P, uint64_t seq, int r) {
  return reinterpret_cast<double*>(sync + sync_slots(P)) +
         ((size_t)(seq % kXRing) * (size_t)P + (size_t)r) * kRecN;
}

// P2P record exchange, step 1: this rank's records seq0 .. seq0+n-1 (its own
// slots) are stored into the same slots of every peer's buffer.
struct XPeers {
  double* slots[kMaxRanks];  // each rank's slot array as mapped here (nullptr: self)
};
__global__ void xpush(const double* mine, XPeers peers, int P, int me, unsigned long long seq0,
                      int n) {
  const int per = n * kRecN;
  for (int i = threadIdx.x; i < P * per; i += blockDim.x) {
    const int q = i / per, k = (i % per) / kRecN, f = i % kRecN;
    if (q == me || !peers.slots[q]) continue;
    const size_t o = ((size_t)((seq0 + (unsigned long long)k) % kXRing) * (size_t)P + me) * kRecN + f;
    peers.slots[q][o] = mine[o];
  }
}

// step 2 (after every peer's signal): the global record of each of the n
// records is the fold of the P ranks' slots in rank order — sums [0..2] added
// 0 + 1 + ... + P-1 left to right, maxima [3..6] — so every rank computes the
// bitwise same value ("each rank sums the slots in rank order").
__global__ void xfold(const double* slots, int P, unsigned long long seq0, int n, double* dst0,
                      double* dst1) {
  const int t = threadIdx.x;
  if (t >= n * kRecN) return;
  const int k = t / kRecN, f = t % kRecN;
  const volatile double* s =
      slots + (size_t)((seq0 + (unsigned long long)k) % kXRing) * (size_t)P * kRecN + f;
  double acc = s[0];
  for (int q = 1; q < P; ++q) {
    const double v = s[(size_t)q * kRecN];
    acc = f < kRecMaxEta ? acc + v : fmax(acc, v);
  }
  (k ? dst1 : dst0)[f] = acc;
}

// NVTX range over an API call (visible in nsys / ncu timelines; ~free
// without a tool attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

int fail(sw2d* h, int code, const std::string& msg) {
  if (h) {
    h->err = msg;
    if (code == SW2D_ECUDA || code == SW2D_ENCCL) h->sticky = code;
  } else {
    t_create_err = msg;
  }
  return code;
}

#define CUDA_TRY(h, call)                                                   \
  do {                                                                      \
    cudaError_t e_ = (call);                                                \
    if (e_ != cudaSuccess)                                                  \
      return fail((h), e_ == cudaErrorMemoryAllocation ? SW2D_ENOMEM        \
                                                       : SW2D_ECUDA,        \
                  std::string(#call) + ": " + cudaGetErrorString(e_));      \
  } while (0)

#define NCCL_TRY(h, call)                                                   \
  do {                                                                      \
    ncclResult_t r_ = (call);                                               \
    if (r_ != ncclSuccess)                                                  \
      return fail((h), SW2D_ENCCL,                                          \
                  std::string(#call) + ": " +                               \
                      sw2d_host::nccl().GetErrorString(r_));                \
  } while (0)

#define ENTER(h)                                                  \
  do {                                                            \
    if (!(h)) return SW2D_EINVAL;                                 \
    if ((h)->sticky) return (h)->sticky;                          \
    CUDA_TRY((h), cudaSetDevice((h)->device));                    \
  } while (0)

bool finite_pos(float x) { return std::isfinite(x) && x > 0.0f; }

int validate(const sw2d_params* p, std::string& why) {
  if (!p) { why = "params is NULL"; return SW2D_EINVAL; }
  if (p->bc != SW2D_BC_CLOSED) { why = "bc must be SW2D_BC_CLOSED"; return SW2D_EUNSUPPORTED; }
  if (p->variant != SW2D_VARIANT_FUSED && p->variant != SW2D_VARIANT_PAPER) {
    why = "unknown variant"; return SW2D_EUNSUPPORTED;
  }
  if (p->nx < 1 || p->ny < 1) { why = "nx, ny must be >= 1"; return SW2D_EINVAL; }
  if (p->nx > (1LL << 30)) { why = "nx too large"; return SW2D_EINVAL; }
  if (!finite_pos(p->dx) || !finite_pos(p->dy) || !finite_pos(p->dt)) {
    why = "dx, dy, dt must be finite and > 0"; return SW2D_EINVAL;
  }
  if (!std::isfinite(p->g) || p->g < 0.0f) { why = "g must be finite and >= 0"; return SW2D_EINVAL; }
  if (!(p->eps >= 0.0f && p->eps <= 1.0f)) { why = "eps must be in [0, 1]"; return SW2D_EINVAL; }
  if (!std::isfinite(p->hmin) || p->hmin < 0.0f) { why = "hmin must be finite and >= 0"; return SW2D_EINVAL; }
  if (p->reduce_every_step >> SW2D_RED_N) { why = "unknown reduction bit"; return SW2D_EINVAL; }
  if (p->history_len < 0) { why = "history_len must be >= 0"; return SW2D_EINVAL; }
  return SW2D_OK;
}

// Coefficients once, in double, one rounding each (reading R12).
Coef make_coef(const sw2d_params& p) {
  Coef c;
  const double t = (double)p.dt * (double)p.g;
  c.cgx = (float)(-(t / (double)p.dx));
  c.cgy = (float)(-(t / (double)p.dy));
  c.cx = (float)((double)p.dt / (double)p.dx);
  c.cy = (float)((double)p.dt / (double)p.dy);
  c.q = 0.25f * p.eps;
  c.hmin = p.hmin;
  c.nz = -0.0f;
  return c;
}

int red_level_of(uint32_t mask) {
  const uint32_t sums = (1u << SW2D_RED_VOLUME) | (1u << SW2D_RED_SUM_ETA);
  if (mask & ~sums) return 2;
  if (mask & sums) return 1;
  return 0;
}

float* fld(float* base, int64_t pitch, int64_t row) { return base + row * pitch; }

// Small grids: the persistent cooperative kernel (sw2d_persist.cu), on one
// GPU without ranks, if its tiles fit co-resident.  By default where it
// measured faster than the graph-replayed row march: up to
// 2^18 cells (C1 1.57 vs 2.62 us/step, C2 3.05 vs 3.68; with VOLUME per step
// 1.92 vs 3.02 and 3.59 vs 4.00); SW2D_PERSIST=0/1 forces it off/on (on: up
// to 2^21 cells).  K = 2 steps per block (SW2D_PERSIST_K); the CTA shape
// (warps x rows per thread; SW2D_PERSIST_SHAPE) minimises the busiest SM's
// work, see below.
constexpr int kPersistRedChunk = 64;   // steps per launch when diagnostics are folded
void plan_persist(sw2d* h) {
  h->pk = 0;
  h->ptag = false;
  const long long cells = h->p.nx * h->p.ny;
  if (h->multi || h->virt || h->p.variant != SW2D_VARIANT_FUSED || h->slabs.size() != 1) return;
  if (cells > kSmallMaxCells) return;
  const char* on = std::getenv("SW2D_PERSIST");
  if (on && std::atoi(on) == 0) return;
  if (!on) {   // the default: where it wins; a forced kernel kind (tests, A/B) wins too
    if (std::getenv("SW2D_STEP_KERNEL")) return;
    if (cells > (1LL << 18)) return;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device);
  int K_force = 0;
  if (const char* e = std::getenv("SW2D_PERSIST_K")) K_force = std::max(1, std::min(4, std::atoi(e)));
  int shape_force = -1;
  if (const char* e = std::getenv("SW2D_PERSIST_SHAPE"))
    shape_force = std::max(0, std::min(persist_shapes() - 1, std::atoi(e)));
  struct Pick { int shape = -1, th = 0, ntx = 0, nty = 0; long long per_sm = 0; double cost = -1; };
  // the shape that minimises the busiest SM's work for K steps per block
  // (ties: the first, more warps)
  auto pick = [&](int K, bool lone_only) {
    Pick best;
    const int tw = persist_tile_cols(K);
    const int ntx = (int)((h->p.nx + tw - 1) / tw);
    for (int sh = 0; sh < persist_shapes(); ++sh) {
      if (shape_force >= 0 && sh != shape_force) continue;
      const int th = persist_tile_rows(K, sh);
      if (th <= 0) continue;
      const int nty = (int)((h->p.ny + th - 1) / th);
      const long long nt = (long long)ntx * nty;
      if (nt > persist_capacity(K, h->red_level, sh)) continue;
      // the busiest SM's shared rows; a lone CTA per SM counted 1.5x (nothing
      // overlaps its handshake), four or more (without the per-step partials'
      // registers) 2/3 (they hide each other's latency).  Measured on C2
      // (profiles/ab_r02q.log): 8 warps x 16 rows, 567 tiles (4 per SM) 3.03
      // us/step, 8 x 24, 288 tiles 3.17 (3.58 vs 3.76 with VOLUME per step);
      // 16 x 32, 189 tiles 3.40; 16 x 48, 117 tiles 3.66.
      const long long per_sm = (nt + sms - 1) / sms;
      if (lone_only && per_sm != 1) continue;
      const double cost = (double)persist_shape_rows(sh) * (double)per_sm *
                          (per_sm == 1 ? 1.5 : 1.0) *
                          (per_sm >= 4 && h->red_level == 0 ? 2.0 / 3.0 : 1.0);
      if (best.cost < 0 || cost < best.cost - 1e-9) {
        best.shape = sh;
        best.th = th;
        best.ntx = ntx;
        best.nty = nty;
        best.per_sm = per_sm;
        best.cost = cost;
      }
    }
    return best;
  };
  // K: 2, or 3 where the K = 2 plan keeps several CTAs on every SM (one
  // handshake per three steps then pays for the wider apron: C2 3.03 -> 2.85
  // us/step with 16 warps x 32 rows; with a lone CTA per SM (C1) the phases'
  // latency dominates and K = 3 is slower, 1.58 -> 2.07).  With per-step
  // partials K = 3 wins only as one 16-warp CTA per SM (C2 VOLUME 3.54 ->
  // 3.43, all 3.78 -> 3.74; as two 16-warp CTAs 3.64: profiles/ab_r02v.log)
  int K = K_force ? K_force : 2;
  Pick p = pick(K, false);
  if (!K_force && p.shape >= 0 && p.per_sm >= 2) {
    const Pick p3 = pick(3, h->red_level > 0);
    if (p3.shape >= 0) {
      K = 3;
      p = p3;
    }
  }
  if (p.shape < 0) return;
  // the handshake: tagged ring words on grids of few tiles (at most one per
  // two SMs: the saved round trip is then the critical path and the polling
  // light, C1 1.56 -> 1.46 us/step); per-tile counters otherwise (C2, 250
  // tiles: 2.82 -> 3.20 tagged; with VOLUME per step, 140 tiles of 48 rows,
  // 3.36 -> 3.52: every apron thread polling strains L2;
  // profiles/ab_r02tagt_handshake.log).  SW2D_PERSIST_TAGGED=0/1 forces.
  h->ptag = 2LL * p.ntx * p.nty <= sms;
  if (const char* e = std::getenv("SW2D_PERSIST_TAGGED")) h->ptag = std::atoi(e) != 0;
  h->pk = K;
  h->pshape = p.shape;
  h->pth = p.th;
  h->pntx = p.ntx;
  h->pnty = p.nty;
}

void plan_launches(sw2d* h) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device);
  int bps = step_occupancy_blocks_per_sm(h->red_level, h->kind);
  if (const char* e = std::getenv("SW2D_CTAS_PER_SM")) bps = std::max(1, std::min(bps, std::atoi(e)));
  long long min_rows = kMinRowsPerSeg;
  if (const char* e = std::getenv("SW2D_MIN_ROWS")) min_rows = std::max(1, std::atoi(e));
  // Rows within kHaloRows of an internal slab boundary read this step's
  // halo (phase 1, after the exchange); the rest (phase 0) overlap with it.
  // Virtual ranks use the same bands, so one GPU exercises the split.
  const char* sk_env = std::getenv("SW2D_SK");
  const bool sk_on = !(sk_env && std::atoi(sk_env) == 0);
  int sk_force = 0;   // SW2D_SK=2: the even split wherever it is possible
  if (sk_env && std::atoi(sk_env) == 2) {
    sk_force = sms;
    if (const char* e = std::getenv("SW2D_SK_CTAS")) sk_force = std::max(1, std::atoi(e));
  }
  auto plan = [&](std::vector<Launch>& out, int per, long long target_segs, long long mrows,
                  int kind, int nstrips) {
    out.clear();
    int part = 0;
    auto add = [&](int s, long long lo, long long hi, int phase) {
      if (hi < lo) return;
      const long long rows = hi - lo + 1;
      long long rps = (rows + target_segs - 1) / target_segs;
      rps = std::max<long long>(rps, mrows);
      Launch L;
      L.slab = s;
      L.row_lo = lo;
      L.row_hi = hi;
      L.rows_per_seg = (int)rps;
      L.nsegs = (int)((rows + rps - 1) / rps);
      L.phase = phase;
      L.blocks = kind == 3 ? (int)(((nstrips + per - 1) / per) * L.nsegs)
                           : step_grid(kind, nstrips, L.nsegs);
      // Two-step CTA kernel: when the column groups x row segments grid does
      // not fill the SMs (C5: 20 groups x 7 segments = 140 of 148), split the
      // group-rows evenly over one CTA per SM instead, if that lowers the
      // busiest CTA's streamed rows (each piece streams 8 extra rows; a share
      // may span two groups).  sms >= 2 x groups keeps a share within two.
      // Real ranks use every SM too: the boundary bands follow the interior
      // launch on the same stream (they need the halo), the P2P transport
      // runs no kernel beside it, and the NCCL exchange kernels (comm stream,
      // highest priority) are dispatched ahead of the interior launch's CTAs
      // when both become ready at the end of the previous pass.
      if (kind == 3 && sk_on) {
        const long long ncc = (nstrips + per - 1) / per;
        const long long skc = sms;
        const long long classic = std::min<long long>(rps, rows) + 8;   // rows per CTA
        const long long even = (rows * ncc + skc - 1) / skc + 2 * 8;
        if (sk_force > 0 && sk_force >= 2 * ncc) {   // tests: SW2D_SK=2 [SW2D_SK_CTAS=n]
          L.sk = sk_force;
          L.blocks = sk_force;
        } else if (sk_force == 0 && L.blocks < skc && skc >= 2 * ncc &&
                   50 * even < 49 * classic) {
          L.sk = (int)skc;
          L.blocks = (int)skc;
        }
      }
      L.part_base = part;
      part += L.blocks;
      out.push_back(L);
    };
    for (int s = 0; s < (int)h->slabs.size(); ++s) {
      const Slab& sl = h->slabs[s];
      const long long J0 = sl.j0 + 1, J1 = sl.j0 + sl.nrows;
      const bool lo_halo = sl.j0 > 0, hi_halo = sl.j0 + sl.nrows < h->p.ny;
      add(s, J0 + (lo_halo ? kHaloRows : 0), J1 - (hi_halo ? kHaloRows : 0), 0);
      if (lo_halo) add(s, J0, J0 + kHaloRows - 1, 1);
      if (hi_halo) add(s, J1 - kHaloRows + 1, J1, 1);
    }
    return part;
  };
  {  // one step per launch
    const int per = step_strips_per_cta(h->kind);
    const long long ncc = (h->nstrips + per - 1) / per;
    h->step_blocks = plan(h->launches, per, std::max(1LL, (long long)sms * bps / ncc), min_rows,
                          h->kind, h->nstrips);
  }
  // two steps per launch (the CTA kernel layout; one CTA per SM)
  h->launches2.clear();
  h->step_blocks2 = 0;
  const char* two_env = std::getenv("SW2D_TWO_STEP");
  const bool two = h->p.variant == SW2D_VARIANT_FUSED && !(two_env && std::atoi(two_env) == 0);
  if (two && h->kind == 1) {
    const int per2 = step2_strips_per_cta();
    const long long ncc2 = (h->nstrips + per2 - 1) / per2;
    h->step_blocks2 = plan(h->launches2, per2, std::max(1LL, (long long)sms / ncc2), 8, 3,
                           h->nstrips);
  } else if (two && h->kind == 2) {  // the small-grid layout, two marches per warp
    const int bps2 = step2_small_occupancy_blocks_per_sm(h->red_level);
    const int per = step_strips_per_cta(2);
    h->nstrips2 = (int)((h->p.nx + step2_small_strip_cols() - 1) / step2_small_strip_cols());
    const long long ncc = (h->nstrips2 + per - 1) / per;
    long long mrows2 = 2;  // min output rows per two-step segment (it streams 8 more; measured)
    if (const char* e = std::getenv("SW2D_MIN_ROWS2")) mrows2 = std::max(1, std::atoi(e));
    h->step_blocks2 = plan(h->launches2, per, std::max(1LL, (long long)sms * bps2 / ncc), mrows2, 2,
                           h->nstrips2);
  }
  plan_persist(h);
  {
    static const char* kinds[] = {"", "cta-ring", "small"};
    std::string split = "grid";   // even-rows:<CTAs> if any two-step launch splits rows
    for (const Launch& L : h->launches2)
      if (L.sk > 0) split = "even-rows:" + std::to_string(L.sk);
    char buf[256];
    std::snprintf(buf, sizeof(buf),
                  "kernel=%s steps_per_launch=%d launches_per_pass=%zu strips=%d "
                  "ctas_per_sm=%d halo=%s split=%s",
                  kinds[h->kind], h->launches2.empty() ? 1 : 2,
                  h->launches2.empty() ? h->launches.size() : h->launches2.size(), h->nstrips,
                  bps, h->halo_mode == SW2D_HALO_P2P ? "p2p" : "nccl", split.c_str());
    h->plan_text = buf;
    if (h->pk) {
      std::snprintf(buf, sizeof(buf),
                    "kernel=persist steps_per_block=%d tiles=%dx%d tile=%dx%d warps=%d "
                    "rows_per_thread=%d handshake=%s cooperative=1 halo=%s",
                    h->pk, h->pntx, h->pnty, persist_tile_cols(h->pk), h->pth,
                    persist_shape_warps(h->pshape),
                    persist_shape_rows(h->pshape) / persist_shape_warps(h->pshape),
                    h->ptag ? "tagged" : "counters",
                    h->halo_mode == SW2D_HALO_P2P ? "p2p" : "nccl");
      h->plan_text = buf;
    }
  }
  if (std::getenv("SW2D_VERBOSE")) {
    std::fprintf(stderr, "[sw2d] kind %d red %d: %d CTAs/SM on %d SMs, %d strips\n", h->kind,
                 h->red_level, bps, sms, h->nstrips);
    for (const Launch& L : h->launches)
      std::fprintf(stderr, "[sw2d]   slab %d rows %lld..%lld phase %d: %d segs x %d rows, %d CTAs\n",
                   L.slab, L.row_lo, L.row_hi, L.phase, L.nsegs, L.rows_per_seg, L.blocks);
    for (const Launch& L : h->launches2)
      std::fprintf(stderr, "[sw2d]   2-step slab %d rows %lld..%lld phase %d: %d segs x %d rows, %d CTAs%s\n",
                   L.slab, L.row_lo, L.row_hi, L.phase, L.nsegs, L.rows_per_seg, L.blocks,
                   L.sk ? " (even split)" : "");
  }
}

StepArgs step_args(sw2d* h, const Launch& L, double* rec) {
  const Slab& sl = h->slabs[L.slab];
  StepArgs a;
  a.s.E = sl.E[h->cur];
  a.s.U = sl.U[h->cur];
  a.s.V = sl.V[h->cur];
  a.s.H0 = sl.H0;
  a.s.En = sl.E[1 - h->cur];
  a.s.Un = sl.U[1 - h->cur];
  a.s.Vn = sl.V[1 - h->cur];
  a.s.pitch = h->pitch;
  a.s.jbase = sl.j0 + 1 - kHaloRows;
  a.s.nelem = (sl.nrows + 2 * kHaloRows) * h->pitch;
  a.nx = (int)h->p.nx;
  a.ny = h->p.ny;
  a.row_lo = L.row_lo;
  a.row_hi = L.row_hi;
  a.rows_per_seg = L.rows_per_seg;
  a.nstrips = h->nstrips;
  a.nsegs = L.nsegs;
  a.sk_ctas = L.sk;
  a.c = h->coef;
  a.red.partials = h->partials;
  a.red.part_base = L.part_base;
  a.red.counter = h->counter;
  a.red.expected = h->step_blocks;
  a.red.rec = rec;
  a.red.h0sum = h->h0sum;
  a.red.dxdy = (double)h->p.dx * (double)h->p.dy;
  return a;
}

// P2P halo mode: the rows of slab L.slab that its neighbours need (its first
// two rows go south, its last two north) are mirrored into their buffers of
// the next state.
void set_remotes(sw2d* h, const Launch& L, StepArgs& a) {
  for (int side = 0; side < 2; ++side) {
    a.rem[side].lo = 1;
    a.rem[side].hi = 0;  // none
  }
  const Slab& sl = h->slabs[L.slab];
  const long long J0 = sl.j0 + 1, J1 = sl.j0 + sl.nrows;
  const int nb = 1 - h->cur;  // the buffer being written this step
  for (int side = 0; side < 2; ++side) {
    float *E = nullptr, *U = nullptr, *V = nullptr;
    long long jb = 0, ne = 0;
    if (h->virt) {
      const int peer = L.slab + (side == 0 ? -1 : 1);
      if (peer < 0 || peer >= (int)h->slabs.size()) continue;
      const Slab& ps = h->slabs[peer];
      E = ps.E[nb]; U = ps.U[nb]; V = ps.V[nb];
      jb = ps.j0 + 1 - kHaloRows;
      ne = (ps.nrows + 2 * kHaloRows) * h->pitch;
    } else {
      const auto& pr = h->nbr[side];
      if (!pr.present) continue;
      E = pr.E[nb]; U = pr.U[nb]; V = pr.V[nb];
      jb = pr.jbase;
      ne = pr.nelem;
    }
    a.rem[side].En = E;
    a.rem[side].Un = U;
    a.rem[side].Vn = V;
    a.rem[side].jbase = jb;
    a.rem[side].nelem = ne;
    a.rem[side].lo = (int)(side == 0 ? J0 : J1 - kHaloRows + 1);
    a.rem[side].hi = (int)(side == 0 ? J0 + kHaloRows - 1 : J1);
  }
}

PaperArgs paper_args(sw2d* h, Slab& sl) {
  PaperArgs a;
  a.E = sl.E[0];
  a.U = sl.U[0];
  a.V = sl.V[0];
  a.H0 = sl.H0;
  a.un = sl.U[1];
  a.vn = sl.V[1];
  a.etan = sl.E[1];
  a.h = sl.Hs;
  a.wet_in = sl.W[h->wcur];
  a.wet_out = sl.W[1 - h->wcur];
  a.Eo = sl.E[0];
  a.Uo = sl.U[0];
  a.Vo = sl.V[0];
  a.pitch = h->pitch;
  a.jbase = sl.j0 + 1 - kHaloRows;
  a.nrows = sl.nrows;
  a.nx = (int)h->p.nx;
  a.ny = h->p.ny;
  a.c = h->coef;
  return a;
}

// Diagnostics of the current state into `rec` with the standalone kernel.
int reduce_into(sw2d* h, double* rec) {
  int expected = 0;
  std::vector<ReduceArgs> ras;
  for (Slab& s : h->slabs) {
    ReduceArgs a{};
    a.E = s.E[h->cur];
    a.U = s.U[h->cur];
    a.V = s.V[h->cur];
    a.H0 = s.H0;
    a.pitch = h->pitch;
    a.nrows = s.nrows;
    a.nx = (int)h->p.nx;
    a.hmin = h->p.hmin;
    a.red.part_base = expected;
    expected += reduce_blocks(a);
    ras.push_back(a);
  }
  for (ReduceArgs& a : ras) {
    a.red.partials = h->partials;
    a.red.counter = h->counter;
    a.red.expected = expected;
    a.red.rec = rec;
    a.red.h0sum = h->h0sum;
    a.red.dxdy = (double)h->p.dx * (double)h->p.dy;
    launch_reduce(a, h->stream);
    h->nlaunch++;
  }
  CUDA_TRY(h, cudaGetLastError());
  return SW2D_OK;
}

// Fields moved by a halo exchange: eta, u, v of buffer b (hzero when b < 0).
int halo_fields(Slab& sl, int b, float** f) {
  if (b < 0) {
    f[0] = sl.H0;
    return 1;
  }
  f[0] = sl.E[b];
  f[1] = sl.U[b];
  f[2] = sl.V[b];
  return 3;
}

// Device copies of the 2-row halos between virtual-rank slabs, following
// sw2d_halo_plan (the same plan the NCCL path runs).
int virtual_halo(sw2d* h, int b) {
  const size_t bytes = (size_t)(kHaloRows * h->pitch) * sizeof(float);
  const int P = (int)h->slabs.size();
  for (int r = 0; r < P; ++r) {
    int64_t plan[4];
    sw2d_halo_plan(h->p.ny, P, r, plan);
    float* mine[3];
    const int nf = halo_fields(h->slabs[r], b, mine);
    for (int side = 0; side < 2; ++side) {  // 0: south neighbour r-1, 1: north r+1
      const int64_t recv_row = plan[2 * side + 1];
      if (recv_row < 0) continue;
      const int peer = side == 0 ? r - 1 : r + 1;
      int64_t pplan[4];
      sw2d_halo_plan(h->p.ny, P, peer, pplan);
      const int64_t send_row = pplan[side == 0 ? 2 : 0];  // what the peer sends towards r
      float* theirs[3];
      halo_fields(h->slabs[peer], b, theirs);
      for (int f = 0; f < nf; ++f)
        CUDA_TRY(h, cudaMemcpyAsync(fld(mine[f], h->pitch, recv_row),
                                    fld(theirs[f], h->pitch, send_row), bytes,
                                    cudaMemcpyDeviceToDevice, h->stream));
    }
  }
  return SW2D_OK;
}

// NCCL exchange of the 2-row halos with the row neighbours following
// sw2d_halo_plan, enqueued on stream `st`.
int nccl_halo(sw2d* h, int b, cudaStream_t st) {
  const auto& nc = sw2d_host::nccl();
  int64_t plan[4];
  sw2d_halo_plan(h->p.ny, h->nranks, h->rank, plan);
  float* f[3];
  const int nf = halo_fields(h->slabs[0], b, f);
  const size_t cnt = (size_t)(kHaloRows * h->pitch);
  NCCL_TRY(h, nc.GroupStart());
  for (int i = 0; i < nf; ++i) {
    for (int side = 0; side < 2; ++side) {
      if (plan[2 * side] < 0) continue;
      const int peer = side == 0 ? h->rank - 1 : h->rank + 1;
      NCCL_TRY(h, nc.Send(fld(f[i], h->pitch, plan[2 * side]), cnt, ncclFloat32, peer,
                          h->comm_nccl, st));
      NCCL_TRY(h, nc.Recv(fld(f[i], h->pitch, plan[2 * side + 1]), cnt, ncclFloat32, peer,
                          h->comm_nccl, st));
    }
  }
  NCCL_TRY(h, nc.GroupEnd());
  return SW2D_OK;
}

// Allreduce of a 7-double record (src -> dst, may alias): sums [0..2], maxima [3..6].
int nccl_allreduce_rec(sw2d* h, const double* src, double* dst, cudaStream_t st) {
  const auto& nc = sw2d_host::nccl();
  NCCL_TRY(h, nc.GroupStart());
  NCCL_TRY(h, nc.AllReduce(src, dst, 3, ncclFloat64, ncclSum, h->comm_nccl, st));
  NCCL_TRY(h, nc.AllReduce(src + 3, dst + 3, 4, ncclFloat64, ncclMax, h->comm_nccl, st));
  NCCL_TRY(h, nc.GroupEnd());
  return SW2D_OK;
}

// Before kernels write this rank's slots of records seq0 .. seq0+n-1 (compute
// stream): the record that last used the newest of those slots has been
// combined (its ev_x was recorded on the comm stream when it was enqueued —
// at least kXRing - 2 records ago, so always recorded already).
int guard_slots(sw2d* h, uint64_t seq0, int n) {
  const uint64_t last = seq0 + (uint64_t)n - 1;
  if (last >= (uint64_t)kXRing)
    CUDA_TRY(h, cudaStreamWaitEvent(h->stream, h->ev_x[(last - kXRing) % kXRing], 0));
  return SW2D_OK;
}

// NCCL mode: allreduce the pending records (slot -> destination) on the comm
// stream, which has already waited for the pass that produced them.
int flush_pending(sw2d* h) {
  for (const sw2d::PendingRec& r : h->pending) {
    int rc = nccl_allreduce_rec(h, xslot(h->sync, h->nranks, r.seq, h->rank), r.dst, h->comm);
    if (rc) return rc;
    CUDA_TRY(h, cudaEventRecord(h->ev_x[r.seq % kXRing], h->comm));
  }
  h->pending.clear();
  return SW2D_OK;
}

// P2P mode: combine records seq0 .. seq0+n-1 (n <= 2; this rank's parts are in
// its own slots) into dst[k] on every rank, on the comm stream (which has
// waited for the work that wrote the slots).  No NCCL: stream memory
// operations order it, kernels move and fold the records.
int p2p_exchange(sw2d* h, uint64_t seq0, int n, double* dst0, double* dst1) {
  const auto& mo = sw2d_host::memops();
  const int P = h->nranks, me = h->rank;
  const uint64_t end = seq0 + (uint64_t)n;
  // 1. every peer has folded the records whose slots these overwrite
  if (end > (uint64_t)kXRing)
    for (int q = 0; q < P; ++q)
      if (q != me && mo.wait32(h->comm, flag_addr(h->sync, sync_xack(P), q),
                               (unsigned)(end - kXRing), 0x0 /*GEQ*/))
        return fail(h, SW2D_ECUDA, "cuStreamWaitValue32 failed");
  // 2. this rank's records into every peer's slots, then tell them
  if (P > 1) {
    XPeers xp{};
    for (int q = 0; q < P; ++q)
      xp.slots[q] = q == me ? nullptr : reinterpret_cast<double*>(h->psync[q] + sync_slots(P));
    xpush<<<1, 128, 0, h->comm>>>(reinterpret_cast<const double*>(h->sync + sync_slots(P)), xp, P,
                                  me, (unsigned long long)seq0, n);
    h->nlaunch++;
    CUDA_TRY(h, cudaGetLastError());
  }
  for (int q = 0; q < P; ++q)
    if (q != me && mo.write32(h->comm, flag_addr(h->psync[q], sync_xflag(), me), (unsigned)end, 0x0))
      return fail(h, SW2D_ECUDA, "cuStreamWriteValue32 failed");
  // 3. every peer's records have landed here
  for (int q = 0; q < P; ++q)
    if (q != me && mo.wait32(h->comm, flag_addr(h->sync, sync_xflag(), q), (unsigned)end, 0x0))
      return fail(h, SW2D_ECUDA, "cuStreamWaitValue32 failed");
  // 4. fold in rank order; the slots are free again once the peers know
  xfold<<<1, 32, 0, h->comm>>>(reinterpret_cast<const double*>(h->sync + sync_slots(P)), P,
                               (unsigned long long)seq0, n, dst0, dst1);
  h->nlaunch++;
  CUDA_TRY(h, cudaGetLastError());
  for (int k = 0; k < n; ++k)
    CUDA_TRY(h, cudaEventRecord(h->ev_x[(seq0 + (uint64_t)k) % kXRing], h->comm));
  for (int q = 0; q < P; ++q)
    if (q != me && mo.write32(h->comm, flag_addr(h->psync[q], sync_xack(P), me), (unsigned)end, 0x0))
      return fail(h, SW2D_ECUDA, "cuStreamWriteValue32 failed");
  return SW2D_OK;
}

double rec_value(const double* rec, int op) {
  switch (op) {
    case SW2D_RED_VOLUME: return rec[kRecVol];
    case SW2D_RED_SUM_ETA: return rec[kRecSumEta];
    case SW2D_RED_MAX_ETA: return rec[kRecMaxEta];
    case SW2D_RED_MIN_ETA: return -rec[kRecNegMinEta];
    case SW2D_RED_MAX_ABS_U: return rec[kRecMaxU];
    case SW2D_RED_MAX_ABS_V: return rec[kRecMaxV];
    default: return rec[kRecWet];
  }
}

void free_all(sw2d* h) {
  for (Slab& s : h->slabs) {
    cudaFree(s.Hs);
    cudaFree(s.W[0]);
    cudaFree(s.W[1]);
    cudaFree(s.H0);
    for (int b = 0; b < 2; ++b) {
      cudaFree(s.E[b]);
      cudaFree(s.U[b]);
      cudaFree(s.V[b]);
    }
  }
  h->slabs.clear();
  cudaFree(h->partials);
  cudaFree(h->counter);
  cudaFree(h->dstep);
  cudaFree(h->grec);
  cudaFree(h->gpart);
  cudaFree(h->hist);
  cudaFree(h->rec);
  cudaFree(h->h0sum);
  cudaFree(h->zero);
  cudaFree(h->bad);
  if (h->bad_host) cudaFreeHost(h->bad_host);
  cudaFree(h->wetbuf);
  cudaFree(h->stage);
  cudaFree(h->snap[0]);
  cudaFree(h->snap[1]);
  for (int b = 0; b < 2; ++b) {
    if (h->ev_snap[b]) cudaEventDestroy(h->ev_snap[b]);
    if (h->ev_copied[b]) cudaEventDestroy(h->ev_copied[b]);
  }
  if (h->copy) cudaStreamDestroy(h->copy);
  if (h->ev_ready) cudaEventDestroy(h->ev_ready);
  if (h->ev_halo) cudaEventDestroy(h->ev_halo);
  if (h->comm) cudaStreamDestroy(h->comm);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  for (auto& pr : h->nbr) {
    for (int b = 0; b < 2; ++b) {
      if (pr.E[b]) cudaIpcCloseMemHandle(pr.E[b]);
      if (pr.U[b]) cudaIpcCloseMemHandle(pr.U[b]);
      if (pr.V[b]) cudaIpcCloseMemHandle(pr.V[b]);
    }
    if (pr.H0) cudaIpcCloseMemHandle(pr.H0);
    pr = sw2d::Peer{};
  }
  for (unsigned char*& q : h->psync) {
    if (q) cudaIpcCloseMemHandle(q);
    q = nullptr;
  }
  cudaFree(h->sync);
  cudaFree(h->pflags);
  cudaFree(h->pring);
  cudaFree(h->ppart);
  for (cudaEvent_t& e : h->ev_x)
    if (e) cudaEventDestroy(e);
  for (int b = 0; b < 2; ++b)
    if (h->graph[b]) cudaGraphExecDestroy(h->graph[b]);
  if (h->comm_nccl && sw2d_host::nccl().ok) sw2d_host::nccl().CommDestroy(h->comm_nccl);
}

// P2P mode across real ranks: this rank's peer blob (sw2d_p2p_export) — the
// geometry the importers check, and the CUDA IPC handles of its six state
// buffers, hzero and the sync buffer.
struct PeerBlob {
  uint32_t magic, version;
  int32_t rank, nranks;
  int64_t nx, ny, pitch, j0, nrows;
  int32_t xring, nhandles;
  cudaIpcMemHandle_t mem[8];  // E0 E1 U0 U1 V0 V1 H0 sync
};
static_assert(sizeof(PeerBlob) <= SW2D_P2P_BLOB_BYTES, "blob size");
constexpr uint32_t kBlobMagic = 0x50325753u;  // "SW2P"

bool p2p_real(const sw2d* h) { return h->multi && h->halo_mode == SW2D_HALO_P2P; }

int p2p_export(sw2d* h, unsigned char* out) {
  if (!p2p_real(h)) return fail(h, SW2D_EINVAL, "sw2d_p2p_export: not a real rank in P2P mode");
  std::memset(out, 0, SW2D_P2P_BLOB_BYTES);
  PeerBlob b{};
  const Slab& sl = h->slabs[0];
  b.magic = kBlobMagic;
  b.version = SW2D_ABI_VERSION;
  b.rank = h->rank;
  b.nranks = h->nranks;
  b.nx = h->p.nx;
  b.ny = h->p.ny;
  b.pitch = h->pitch;
  b.j0 = sl.j0;
  b.nrows = sl.nrows;
  b.xring = kXRing;
  b.nhandles = 8;
  void* mine[8] = {sl.E[0], sl.E[1], sl.U[0], sl.U[1], sl.V[0], sl.V[1], sl.H0, h->sync};
  for (int i = 0; i < 8; ++i) CUDA_TRY(h, cudaIpcGetMemHandle(&b.mem[i], mine[i]));
  std::memcpy(out, &b, sizeof(b));
  return SW2D_OK;
}

// Map the peers from all ranks' blobs (rank order): the row neighbours' state
// buffers and hzero (halo stores) and every peer's sync buffer (flags, slots).
int p2p_import(sw2d* h, const unsigned char* blobs) {
  if (!p2p_real(h)) return fail(h, SW2D_EINVAL, "sw2d_p2p_import: not a real rank in P2P mode");
  if (h->p2p_ready) return fail(h, SW2D_EINVAL, "sw2d_p2p_import: peers already mapped");
  if (!sw2d_host::memops().ok)
    return fail(h, SW2D_EUNSUPPORTED, "cuStreamWaitValue32/WriteValue32 unavailable");
  std::vector<PeerBlob> bs((size_t)h->nranks);
  for (int q = 0; q < h->nranks; ++q) {
    std::memcpy(&bs[q], blobs + (size_t)q * SW2D_P2P_BLOB_BYTES, sizeof(PeerBlob));
    const PeerBlob& b = bs[q];
    int64_t j0 = 0, nrows = 0;
    sw2d_partition(h->p.ny, h->nranks, q, &j0, &nrows);
    if (b.magic != kBlobMagic || b.version != SW2D_ABI_VERSION || b.rank != q ||
        b.nranks != h->nranks || b.nx != h->p.nx || b.ny != h->p.ny || b.pitch != h->pitch ||
        b.j0 != j0 || b.nrows != nrows || b.xring != kXRing || b.nhandles != 8)
      return fail(h, SW2D_EINVAL,
                  "sw2d_p2p_import: blob " + std::to_string(q) +
                      " does not match this grid / partition / rank order / library");
  }
  h->psync.assign((size_t)h->nranks, nullptr);
  for (int q = 0; q < h->nranks; ++q) {
    if (q == h->rank) continue;
    void* p = nullptr;
    CUDA_TRY(h, cudaIpcOpenMemHandle(&p, bs[q].mem[7], cudaIpcMemLazyEnablePeerAccess));
    h->psync[q] = (unsigned char*)p;
  }
  for (int side = 0; side < 2; ++side) {
    const int q = side == 0 ? h->rank - 1 : h->rank + 1;
    if (q < 0 || q >= h->nranks) continue;
    auto& pr = h->nbr[side];
    void* p[7];
    for (int i = 0; i < 7; ++i) {
      CUDA_TRY(h, cudaIpcOpenMemHandle(&p[i], bs[q].mem[i], cudaIpcMemLazyEnablePeerAccess));
      switch (i) {  // recorded one by one so free_all closes what was opened
        case 0: pr.E[0] = (float*)p[i]; break;
        case 1: pr.E[1] = (float*)p[i]; break;
        case 2: pr.U[0] = (float*)p[i]; break;
        case 3: pr.U[1] = (float*)p[i]; break;
        case 4: pr.V[0] = (float*)p[i]; break;
        case 5: pr.V[1] = (float*)p[i]; break;
        default: pr.H0 = (float*)p[i]; break;
      }
    }
    pr.jbase = bs[q].j0 + 1 - kHaloRows;
    pr.nrows = bs[q].nrows;
    pr.nelem = (bs[q].nrows + 2 * kHaloRows) * h->pitch;
    pr.present = true;
  }
  h->p2p_ready = true;
  return SW2D_OK;
}

// P2P with an NCCL bootstrap: the blobs travel by one NCCL all-gather at create.
int setup_p2p_nccl(sw2d* h) {
  const auto& nc = sw2d_host::nccl();
  const size_t per = SW2D_P2P_BLOB_BYTES;
  std::vector<unsigned char> mine(per), all(per * (size_t)h->nranks);
  int rc = p2p_export(h, mine.data());
  if (rc) return rc;
  unsigned char* dsend = nullptr;
  unsigned char* drecv = nullptr;
  CUDA_TRY(h, cudaMalloc(&dsend, per));
  CUDA_TRY(h, cudaMalloc(&drecv, per * (size_t)h->nranks));
  CUDA_TRY(h, cudaMemcpy(dsend, mine.data(), per, cudaMemcpyHostToDevice));
  NCCL_TRY(h, nc.AllGather(dsend, drecv, per, ncclUint8, h->comm_nccl, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  CUDA_TRY(h, cudaMemcpy(all.data(), drecv, all.size(), cudaMemcpyDeviceToHost));
  cudaFree(dsend);
  cudaFree(drecv);
  return p2p_import(h, all.data());
}

// P2P mode, in sw2d_set_state: once each neighbour has finished every pass it
// was given (its signals so far have arrived: it no longer reads its halos),
// store this rank's boundary rows of hzero and of state 0 into its halo rows,
// then signal it.  The first pass waits for that signal.
int p2p_halo_init(sw2d* h) {
  const auto& mo = sw2d_host::memops();
  int64_t plan[4];
  sw2d_halo_plan(h->p.ny, h->nranks, h->rank, plan);
  Slab& sl = h->slabs[0];
  const size_t bytes = (size_t)(kHaloRows * h->pitch) * sizeof(float);
  for (int side = 0; side < 2; ++side) {
    const auto& pr = h->nbr[side];
    if (!pr.present) continue;
    if (mo.wait32(h->stream, flag_addr(h->sync, 0, side), h->hseq, 0x0))
      return fail(h, SW2D_ECUDA, "cuStreamWaitValue32 failed");
    // rows this rank sends towards `side` land in the neighbour's halo facing us:
    // its north halo (storage rows nrows+4..) for the south neighbour, its
    // south halo (rows 0..3) for the north one
    const int64_t send_row = plan[2 * side];
    const int64_t recv_row = side == 0 ? pr.nrows + kHaloRows : 0;
    const float* src[4] = {sl.H0, sl.E[0], sl.U[0], sl.V[0]};
    float* dst[4] = {pr.H0, pr.E[0], pr.U[0], pr.V[0]};
    for (int f = 0; f < 4; ++f)
      CUDA_TRY(h, cudaMemcpyAsync(fld(dst[f], h->pitch, recv_row), fld((float*)src[f], h->pitch, send_row),
                                  bytes, cudaMemcpyDeviceToDevice, h->stream));
  }
  for (int side = 0; side < 2; ++side)
    if (h->nbr[side].present &&
        mo.write32(h->stream, flag_addr(h->psync[h->rank + (side ? 1 : -1)], 0, 1 - side),
                   h->hseq + 1, 0x0))
      return fail(h, SW2D_ECUDA, "cuStreamWriteValue32 failed");
  h->hseq++;
  return SW2D_OK;
}

int create_impl(sw2d* h, const sw2d_params* params, const sw2d_dist* dist,
                void* cuda_stream) {
  h->p = *params;
  if (h->p.history_len == 0) h->p.history_len = kDefaultHistory;
  h->coef = make_coef(h->p);
  h->red_level = red_level_of(h->p.reduce_every_step);
  if (const char* e = std::getenv("SW2D_MIN_RED")) h->red_level = std::max(h->red_level, std::atoi(e));
  h->hist_len = h->p.history_len;
  if (dist) {
    if (dist->nranks < 1 || dist->rank < 0 || dist->rank >= dist->nranks)
      return fail(h, SW2D_EINVAL, "bad rank / nranks");
    h->rank = dist->rank;
    h->nranks = dist->nranks;
    h->virt = dist->virtual_ranks != 0;
    // SW2D_FORCE_NCCL=1 (tests): a single real rank still runs the NCCL
    // machinery (communicator, comm stream, grouped exchange with no peers,
    // per-step allreduces), so one GPU exercises that path end to end
    const char* fe = std::getenv("SW2D_FORCE_NCCL");
    h->multi = !h->virt && (h->nranks > 1 || (fe && std::atoi(fe) != 0));
    if (dist->halo_mode != SW2D_HALO_NCCL && dist->halo_mode != SW2D_HALO_P2P)
      return fail(h, SW2D_EINVAL, "unknown halo_mode");
    h->halo_mode = dist->halo_mode;
    if (dist->bootstrap != SW2D_BOOT_NCCL && dist->bootstrap != SW2D_BOOT_EXTERNAL)
      return fail(h, SW2D_EINVAL, "unknown bootstrap");
    h->bootstrap = dist->bootstrap;
    if (h->multi && h->bootstrap == SW2D_BOOT_EXTERNAL && h->halo_mode != SW2D_HALO_P2P)
      return fail(h, SW2D_EINVAL, "SW2D_BOOT_EXTERNAL needs SW2D_HALO_P2P");
    if (h->multi && h->nranks > kMaxRanks)
      return fail(h, SW2D_EUNSUPPORTED, "more than 128 real ranks");
    if (dist->device >= 0) CUDA_TRY(h, cudaSetDevice(dist->device));
  }
  CUDA_TRY(h, cudaGetDevice(&h->device));
  if (h->p.variant == SW2D_VARIANT_PAPER && h->nranks > 1)
    return fail(h, SW2D_EUNSUPPORTED, "the paper variant runs on one GPU without ranks");
  // slabs
  if (h->virt) {
    for (int r = 0; r < h->nranks; ++r) {
      Slab s;
      if (sw2d_partition(h->p.ny, h->nranks, r, &s.j0, &s.nrows) != SW2D_OK)
        return fail(h, SW2D_EINVAL, "ny too small for nranks (need >= 8 rows per rank)");
      h->slabs.push_back(s);
    }
  } else {
    Slab s;
    if (sw2d_partition(h->p.ny, h->nranks, h->rank, &s.j0, &s.nrows) != SW2D_OK)
      return fail(h, SW2D_EINVAL, "ny too small for nranks (need >= 8 rows per rank)");
    h->slabs.push_back(s);
  }
  // kernel kind: the CTA/TMA kernel, or the small-grid kernel for grids that
  // are L2-resident and latency-bound (SW2D_STEP_KERNEL overrides)
  if (h->halo_mode != SW2D_HALO_P2P && h->p.nx * h->p.ny <= kSmallMaxCells) h->kind = 2;
  if (const char* k = std::getenv("SW2D_STEP_KERNEL")) {
    const int v = std::atoi(k);
    h->kind = v == 2 ? 2 : 1;
  }
  if (h->halo_mode == SW2D_HALO_P2P) h->kind = 1;  // the fused halo lives in the CTA kernel
  if (const char* e = std::getenv("SW2D_FAULT_SKIP_HALO")) h->fault_skip_halo = std::atoll(e);
  const int64_t strips4 = (h->p.nx + kColsPerStrip - 1) / kColsPerStrip;
  h->nstrips = (int)((h->p.nx + step_strip_cols(h->kind) - 1) / step_strip_cols(h->kind));
  // storage columns touched: 120-column strips (kinds 0, 1; the 60-column
  // small-grid strips fit inside) and the 56-column two-step small strips
  const int64_t strips56 = (h->p.nx + step2_small_strip_cols() - 1) / step2_small_strip_cols();
  const int64_t need = std::max<int64_t>(strips4 * kColsPerStrip + kStripBase + 8,
                                         strips56 * step2_small_strip_cols() + kColOff + 5);
  h->pitch = (need + 31) / 32 * 32;
  // streams
  if (cuda_stream) {
    h->stream = (cudaStream_t)cuda_stream;
  } else {
    CUDA_TRY(h, cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    h->own_stream = true;
  }
  CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_ready, cudaEventDisableTiming));
  CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_halo, cudaEventDisableTiming));
  if (h->multi) {  // the comm stream's small kernels go ahead of pending step CTAs
    int lo = 0, hi = 0;
    CUDA_TRY(h, cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CUDA_TRY(h, cudaStreamCreateWithPriority(&h->comm, cudaStreamNonBlocking, hi));
  }
  // fields: (nrows + 4) x pitch floats each, zeroed (halo rows / columns stay 0)
  for (Slab& s : h->slabs) {
    const size_t bytes = (size_t)(s.nrows + 2 * kHaloRows) * (size_t)h->pitch * sizeof(float);
    float** all[7] = {&s.H0, &s.E[0], &s.E[1], &s.U[0], &s.U[1], &s.V[0], &s.V[1]};
    for (float** f : all) {
      CUDA_TRY(h, cudaMalloc(f, bytes));
      CUDA_TRY(h, cudaMemsetAsync(*f, 0, bytes, h->stream));
    }
    if (h->p.variant == SW2D_VARIANT_PAPER) {
      const size_t wbytes = (size_t)(s.nrows + 2 * kHaloRows) * (size_t)h->pitch;
      CUDA_TRY(h, cudaMalloc(&s.Hs, bytes));
      CUDA_TRY(h, cudaMemsetAsync(s.Hs, 0, bytes, h->stream));
      for (int b = 0; b < 2; ++b) {
        CUDA_TRY(h, cudaMalloc(&s.W[b], wbytes));
        CUDA_TRY(h, cudaMemsetAsync(s.W[b], 0, wbytes, h->stream));
      }
    }
  }
  plan_launches(h);
  if (h->pk) {
    const size_t nt = (size_t)h->pntx * (size_t)h->pnty;
    const size_t fw = persist_flag_words((int)nt);
    CUDA_TRY(h, cudaMalloc(&h->pflags, fw * sizeof(unsigned)));
    CUDA_TRY(h, cudaMemsetAsync(h->pflags, 0, fw * sizeof(unsigned), h->stream));
    if (h->ptag) {   // tags start at 0: never a block's (its tag >= 1)
      const size_t rw = persist_ring_words(h->p.nx, h->p.ny);
      CUDA_TRY(h, cudaMalloc(&h->pring, rw * sizeof(unsigned long long)));
      CUDA_TRY(h, cudaMemsetAsync(h->pring, 0, rw * sizeof(unsigned long long), h->stream));
    }
    CUDA_TRY(h, cudaMalloc(&h->ppart, nt * (size_t)persist_shape_warps(h->pshape) *
                                          kPersistRedChunk * sizeof(RedPartial)));
  }
  // reduction scratch
  long long cap = std::max<long long>(h->step_blocks, 2LL * h->step_blocks2);
  for (const Slab& s : h->slabs) {
    IngestArgs ia{};
    ia.nrows = s.nrows;
    ia.nx = (int)h->p.nx;
    ReduceArgs ra{};
    ra.nrows = s.nrows;
    ra.nx = (int)h->p.nx;
    cap = std::max<long long>(cap, (long long)ingest_blocks(ia) * (long long)h->slabs.size());
    cap = std::max<long long>(cap, (long long)reduce_blocks(ra) * (long long)h->slabs.size());
  }
  h->partials_cap = (int)cap;
  CUDA_TRY(h, cudaMalloc(&h->partials, sizeof(RedPartial) * (size_t)cap));
  CUDA_TRY(h, cudaMalloc(&h->counter, 2 * sizeof(unsigned int)));
  CUDA_TRY(h, cudaMalloc(&h->dstep, sizeof(unsigned long long)));
  CUDA_TRY(h, cudaMalloc(&h->grec, sizeof(double) * kRecN * 2 * (size_t)kGraphPasses));
  CUDA_TRY(h, cudaMalloc(&h->gpart, sizeof(RedPartial) * (size_t)cap * 2 * (size_t)kGraphPasses));
  CUDA_TRY(h, cudaMemsetAsync(h->counter, 0, 2 * sizeof(unsigned int), h->stream));
  CUDA_TRY(h, cudaMalloc(&h->hist, sizeof(double) * kRecN * (size_t)h->hist_len));
  CUDA_TRY(h, cudaMemsetAsync(h->hist, 0, sizeof(double) * kRecN * (size_t)h->hist_len, h->stream));
  // scratch: up to 2 steps' records, plus a discard record
  CUDA_TRY(h, cudaMalloc(&h->rec, 3 * sizeof(double) * kRecN));
  CUDA_TRY(h, cudaMalloc(&h->h0sum, sizeof(double)));
  CUDA_TRY(h, cudaMalloc(&h->zero, sizeof(double)));
  CUDA_TRY(h, cudaMemsetAsync(h->zero, 0, sizeof(double), h->stream));
  CUDA_TRY(h, cudaMemsetAsync(h->h0sum, 0, sizeof(double), h->stream));
  CUDA_TRY(h, cudaMalloc(&h->bad, sizeof(int)));
  CUDA_TRY(h, cudaHostAlloc(&h->bad_host, sizeof(int), cudaHostAllocMapped));
  // real ranks: the sync buffer (flags, record slots), then the NCCL
  // communicator (SW2D_BOOT_NCCL), which in P2P mode only all-gathers the blobs
  if (h->multi) {
    h->sync_bytes = sync_size(h->nranks);
    CUDA_TRY(h, cudaMalloc(&h->sync, h->sync_bytes));
    CUDA_TRY(h, cudaMemsetAsync(h->sync, 0, h->sync_bytes, h->stream));
    for (cudaEvent_t& e : h->ev_x) CUDA_TRY(h, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    h->psync.assign((size_t)h->nranks, nullptr);
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    if (h->bootstrap == SW2D_BOOT_NCCL) {
      const auto& nc = sw2d_host::nccl();
      if (!nc.ok) return fail(h, SW2D_ENCCL, std::string("NCCL unavailable: ") + nc.why);
      ncclUniqueId id;
      std::memcpy(id.internal, dist->nccl_id, sizeof(id.internal));
      NCCL_TRY(h, nc.CommInitRank(&h->comm_nccl, h->nranks, id, h->rank));
      if (h->halo_mode == SW2D_HALO_P2P) {
        int rc = setup_p2p_nccl(h);
        if (rc) return rc;
      }
    }
  }
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  return SW2D_OK;
}

// One pass of `spl` (1 or 2) model steps over every slab this handle holds:
// the pass's halo exchange (device copies for virtual ranks, NCCL on the comm
// stream, or in P2P mode a wait on the neighbours' flags), the interior
// launches (phase 0, overlapping the exchange), the boundary launches
// (phase 1; in P2P mode they also store their rows into the neighbours'
// halos), the neighbours' signal, and the per-step diagnostics' allreduce.
__global__ void set_dstep(unsigned long long* dstep, unsigned long long v) { *dstep = v; }

// end of a replayed graph: its n records go to history slots (*dstep + i) % len
__global__ void ring_scatter(const double* grec, double* hist, int len,
                             unsigned long long* dstep, int n) {
  const unsigned long long s0 = *dstep;
  const int first = n > len ? n - len : 0;  // earlier records would be overwritten
  for (int t = first * kRecN + threadIdx.x; t < n * kRecN; t += blockDim.x) {
    const int i = t / kRecN, f = t % kRecN;
    hist[(size_t)((s0 + (unsigned long long)i) % (unsigned long long)len) * kRecN + f] = grec[t];
  }
  __syncthreads();
  if (threadIdx.x == 0) *dstep = s0 + (unsigned long long)n;
}

__global__ void publish_word(const int* src, int* dst_host_mapped) {
  *(volatile int*)dst_host_mapped = *src;
}

// 2D copy between a dense [rows][nx] array and the pitched field layout (the
// device side of host transfers: the host side is one contiguous DMA per
// field, which runs at full PCIe rate in both directions at once — pitched
// cudaMemcpy2DAsync transfers did not overlap with each other)
__global__ void copy_rows(float* dst, long long dpitch, const float* src, long long spitch,
                          long long nrows, int nx) {
  const long long n = nrows * (long long)nx;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / nx, c = i - r * nx;
    dst[r * dpitch + c] = src[r * spitch + c];
  }
}

void launch_copy_rows(sw2d* h, float* dst, long long dpitch, const float* src, long long spitch,
                      long long nrows) {
  const long long n = nrows * h->p.nx;
  if (n <= 0) return;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * 16);
  copy_rows<<<blocks, 256, 0, h->stream>>>(dst, dpitch, src, spitch, nrows, (int)h->p.nx);
  h->nlaunch++;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// dense staging for `fields` fields of the handle's rows
int ensure_stage(sw2d* h, int fields, int64_t rows) {
  const size_t need = (size_t)fields * (size_t)rows * (size_t)h->p.nx;
  if (need <= h->stage_floats) return SW2D_OK;
  cudaFree(h->stage);
  h->stage = nullptr;
  h->stage_floats = 0;
  CUDA_TRY(h, cudaMalloc(&h->stage, need * sizeof(float)));
  h->stage_floats = need;
  return SW2D_OK;
}

int run_pass(sw2d* h, int spl) {
  const bool p2p = h->halo_mode == SW2D_HALO_P2P && (h->virt || h->multi);
  const auto& mo = sw2d_host::memops();
  const std::vector<Launch>& launches = spl == 2 ? h->launches2 : h->launches;
  const int blocks = spl == 2 ? h->step_blocks2 : h->step_blocks;
  // dst: where each step's (global) record ends up; rec: where the kernels
  // write it — the same, or with real ranks this rank's exchange slot
  const bool xrec = h->multi && h->red_level;
  double* rec[2];
  double* dst[2];
  for (int k = 0; k < 2; ++k) {
    dst[k] = !h->red_level ? h->rec + k * kRecN
             : h->capturing ? h->grec + (size_t)(h->cap_step + k) * kRecN
                            : h->hist + (size_t)((h->steps + k) % h->hist_len) * kRecN;
    rec[k] = xrec ? xslot(h->sync, h->nranks, h->xseq + (uint64_t)k, h->rank) : dst[k];
  }
  // a one-record ring keeps only the pass's second record (two writers of one
  // slot would race): the first goes to a discard record
  if (spl == 2 && h->red_level && !h->capturing && h->hist_len == 1) {
    dst[0] = h->rec + 2 * kRecN;
    if (!xrec) rec[0] = dst[0];
  }
  if (xrec) {
    int rc = guard_slots(h, h->xseq, spl);
    if (rc) return rc;
  }
  // captured two-step small-grid passes defer their diagnostics: CTA partials
  // go to gpart[step within the graph], folded by fold_steps at the graph's end
  const bool defer = h->capturing && h->red_level && spl == 2 && h->kind == 2;
  const int cap0 = h->cap_step;
  if (h->capturing) h->cap_step += spl;
  // fault injection (tests of the tests): SW2D_FAULT_SKIP_HALO=k drops the
  // halo exchange of the pass that starts step k
  const bool skip_halo = h->fault_skip_halo >= 0 && h->fault_skip_halo >= h->steps &&
                         h->fault_skip_halo < h->steps + spl;
  if (h->virt && !p2p && !skip_halo) {
    int rc = virtual_halo(h, h->cur);
    if (rc) return rc;
  }
  if (h->multi && !p2p) {
    CUDA_TRY(h, cudaStreamWaitEvent(h->comm, h->ev_ready, 0));
    int rc = nccl_halo(h, h->cur, h->comm);
    if (rc) return rc;
    CUDA_TRY(h, cudaEventRecord(h->ev_halo, h->comm));
    rc = flush_pending(h);  // the previous pass's diagnostics, behind the exchange
    if (rc) return rc;
  }
  auto args = [&](const Launch& L) {
    StepArgs a = step_args(h, L, rec[0]);
    if (spl == 2 && h->kind == 2) a.nstrips = h->nstrips2;  // 56-column two-step strips
    a.red.expected = blocks;
    a.red2 = a.red;
    a.red2.partials = h->partials + blocks;
    a.red2.counter = h->counter + 1;
    a.red2.rec = rec[1];
    if (defer) {
      a.red.partials = h->gpart + (size_t)cap0 * (size_t)blocks;
      a.red2.partials = h->gpart + (size_t)(cap0 + 1) * (size_t)blocks;
    }
    return a;
  };
  auto launch = [&](const StepArgs& a, bool remote) {
    if (spl == 2 && h->kind == 2)
      launch_step2_small(a, h->red_level, h->stream, defer);
    else if (spl == 2)
      launch_step2(a, h->red_level, h->stream, remote);
    else
      launch_step(a, h->red_level, h->kind, h->stream, remote);
    h->nlaunch++;
  };
  for (const Launch& L : launches)
    if (L.phase == 0) launch(args(L), false);
  bool any1 = false;
  for (const Launch& L : launches) any1 |= L.phase == 1;
  if (any1 && h->multi) {
    if (p2p) {
      // every signal sent to us so far has arrived: the neighbour's previous
      // pass (or its set_state) has stored our halo rows and no longer reads
      // its own halo rows of the buffer this pass writes
      for (int side = 0; side < 2; ++side)
        if (h->nbr[side].present &&
            mo.wait32(h->stream, flag_addr(h->sync, 0, side), h->hseq, 0x0 /*GEQ*/))
          return fail(h, SW2D_ECUDA, "cuStreamWaitValue32 failed");
    } else {
      CUDA_TRY(h, cudaStreamWaitEvent(h->stream, h->ev_halo, 0));
    }
  }
  for (const Launch& L : launches)
    if (L.phase == 1) {
      StepArgs a = args(L);
      if (p2p) set_remotes(h, L, a);
      launch(a, p2p);
    }
  CUDA_TRY(h, cudaGetLastError());
  if (h->multi) {
    if (p2p) {  // tell the neighbours this pass's rows have landed in their halos
      for (int side = 0; side < 2; ++side)
        if (h->nbr[side].present &&
            mo.write32(h->stream, flag_addr(h->psync[h->rank + (side ? 1 : -1)], 0, 1 - side),
                       h->hseq + 1, 0x0))
          return fail(h, SW2D_ECUDA, "cuStreamWriteValue32 failed");
      h->hseq++;
    }
    CUDA_TRY(h, cudaEventRecord(h->ev_ready, h->stream));
    if (xrec) {
      if (p2p) {
        CUDA_TRY(h, cudaStreamWaitEvent(h->comm, h->ev_ready, 0));
        int rc = p2p_exchange(h, h->xseq, spl, dst[0], dst[1]);
        if (rc) return rc;
      } else {
        for (int k = 0; k < spl; ++k) h->pending.push_back({h->xseq + (uint64_t)k, dst[k]});
      }
      h->xseq += (uint64_t)spl;
    }
  }
  h->cur = 1 - h->cur;
  h->steps += spl;
  return SW2D_OK;
}

}  // namespace

extern "C" {

int sw2d_abi_version(void) { return SW2D_ABI_VERSION; }

int sw2d_partition(int64_t ny, int32_t nranks, int32_t rank, int64_t* j0,
                   int64_t* nrows) {
  if (!j0 || !nrows || nranks < 1 || rank < 0 || rank >= nranks || ny < 1)
    return SW2D_EINVAL;
  const int64_t base = ny / nranks, rem = ny % nranks;
  const int64_t n = base + (rank < rem ? 1 : 0);
  if (nranks > 1 && base < 2 * kHaloRows) return SW2D_EINVAL;  // the smallest slab
  *j0 = (int64_t)rank * base + std::min<int64_t>(rank, rem);
  *nrows = n;
  return SW2D_OK;
}

int sw2d_halo_plan(int64_t ny, int32_t nranks, int32_t rank, int64_t out[4]) {
  int64_t j0, nrows;
  if (!out) return SW2D_EINVAL;
  const int rc = sw2d_partition(ny, nranks, rank, &j0, &nrows);
  if (rc != SW2D_OK) return rc;
  // storage rows: 0,1 south halo | 2 .. nrows+1 owned | nrows+2, nrows+3 north halo
  const bool south = rank > 0, north = rank < nranks - 1;
  out[0] = south ? kHaloRows : -1;           // first owned rows -> south neighbour
  out[1] = south ? 0 : -1;                   // its last owned rows -> south halo
  out[2] = north ? nrows : -1;               // last owned rows -> north neighbour
  out[3] = north ? nrows + kHaloRows : -1;   // its first owned rows -> north halo
  return (south ? 1 : 0) + (north ? 1 : 0);
}

int sw2d_nccl_unique_id(unsigned char out[128]) {
  if (!out) return SW2D_EINVAL;
  const auto& nc = sw2d_host::nccl();
  if (!nc.ok) {
    t_create_err = std::string("NCCL unavailable: ") + nc.why;
    return SW2D_ENCCL;
  }
  ncclUniqueId id;
  if (nc.GetUniqueId(&id) != ncclSuccess) {
    t_create_err = "ncclGetUniqueId failed";
    return SW2D_ENCCL;
  }
  std::memcpy(out, id.internal, sizeof(id.internal));
  return SW2D_OK;
}

int sw2d_create(const sw2d_params* params, const sw2d_dist* dist,
                void* cuda_stream, sw2d** out) {
  if (!out) return SW2D_EINVAL;
  *out = nullptr;
  std::string why;
  const int v = validate(params, why);
  if (v != SW2D_OK) return fail(nullptr, v, why);
  sw2d* h = new (std::nothrow) sw2d();
  if (!h) return fail(nullptr, SW2D_ENOMEM, "host allocation failed");
  const int rc = create_impl(h, params, dist, cuda_stream);
  if (rc != SW2D_OK) {
    t_create_err = h->err;
    free_all(h);
    delete h;
    return rc;
  }
  *out = h;
  return SW2D_OK;
}

int sw2d_p2p_export(sw2d* h, void* out, size_t cap) {
  NvtxRange nvtx_("sw2d_p2p_export");
  ENTER(h);
  if (!out || cap < SW2D_P2P_BLOB_BYTES)
    return fail(h, SW2D_EINVAL, "sw2d_p2p_export: out needs SW2D_P2P_BLOB_BYTES");
  return p2p_export(h, (unsigned char*)out);
}

int sw2d_p2p_import(sw2d* h, const void* blobs, size_t nbytes) {
  NvtxRange nvtx_("sw2d_p2p_import");
  ENTER(h);
  if (!blobs || nbytes != (size_t)SW2D_P2P_BLOB_BYTES * (size_t)h->nranks)
    return fail(h, SW2D_EINVAL, "sw2d_p2p_import: need nranks * SW2D_P2P_BLOB_BYTES bytes");
  return p2p_import(h, (const unsigned char*)blobs);
}

int sw2d_local_rows(const sw2d* h, int64_t* j0, int64_t* nrows) {
  if (!h || !j0 || !nrows) return SW2D_EINVAL;
  *j0 = h->slabs.front().j0;
  *nrows = h->slabs.back().j0 + h->slabs.back().nrows - h->slabs.front().j0;
  return SW2D_OK;
}

int sw2d_local_shape(const sw2d* h, int64_t* nrows, int64_t* nx) {
  int64_t j0 = 0;
  const int rc = sw2d_local_rows(h, &j0, nrows);
  if (rc != SW2D_OK || !nx) return SW2D_EINVAL;
  *nx = h->p.nx;
  return SW2D_OK;
}

int sw2d_set_state(sw2d* h, const float* hzero, const float* eta,
                   const float* u, const float* v) {
  NvtxRange nvtx_("sw2d_set_state");
  ENTER(h);
  if (!hzero || !eta) return fail(h, SW2D_EINVAL, "hzero and eta are required");
  if (p2p_real(h) && !h->p2p_ready)
    return fail(h, SW2D_ESTATE, "P2P ranks: sw2d_p2p_import before sw2d_set_state");
  const int64_t nx = h->p.nx, hj0 = h->slabs.front().j0;
  const size_t wbytes = (size_t)nx * sizeof(float);
  const size_t dp = (size_t)h->pitch * sizeof(float);
  int64_t rows = 0;
  for (Slab& s : h->slabs) rows += s.nrows;
  const size_t cells = (size_t)rows * (size_t)nx;
  CUDA_TRY(h, cudaMemsetAsync(h->bad, 0, sizeof(int), h->stream));
  const float* src[4] = {hzero, eta, u, v};
  // host arrays: one contiguous DMA per field into the dense stage, then a
  // device copy into the pitched fields; device arrays: the device copy alone
  const float* dense[4] = {nullptr, nullptr, nullptr, nullptr};
  for (int f = 0; f < 4; ++f) {
    if (!src[f]) continue;
    if (is_device_ptr(src[f])) {
      dense[f] = src[f];
      continue;
    }
    int rc = ensure_stage(h, 4, rows);
    if (rc) return rc;
    float* st = h->stage + (size_t)f * cells;
    CUDA_TRY(h, cudaMemcpyAsync(st, src[f], cells * sizeof(float), cudaMemcpyHostToDevice,
                                h->stream));
    dense[f] = st;
  }
  for (Slab& s : h->slabs) {
    const size_t src_off = (size_t)(s.j0 - hj0) * (size_t)nx;
    float* dst[4] = {s.H0, s.E[0], s.U[0], s.V[0]};
    for (int f = 0; f < 4; ++f) {
      float* d = dst[f] + kHaloRows * h->pitch + 1 + kColOff;
      if (dense[f])
        launch_copy_rows(h, d, h->pitch, dense[f] + src_off, nx, s.nrows);
      else
        CUDA_TRY(h, cudaMemset2DAsync(d, dp, 0, wbytes, (size_t)s.nrows, h->stream));
    }
  }
  CUDA_TRY(h, cudaGetLastError());
  // finiteness, wall faces, sum(hzero) — one fold over all slabs
  int expected = 0;
  std::vector<IngestArgs> ias;
  for (Slab& s : h->slabs) {
    IngestArgs a{};
    a.E = s.E[0];
    a.U = s.U[0];
    a.V = s.V[0];
    a.H0 = s.H0;
    a.pitch = h->pitch;
    a.jbase = s.j0 + 1 - kHaloRows;
    a.nrows = s.nrows;
    a.nx = (int)nx;
    a.ny = h->p.ny;
    a.bad = h->bad;
    a.red.part_base = expected;
    expected += ingest_blocks(a);
    ias.push_back(a);
  }
  for (IngestArgs& a : ias) {
    a.red.partials = h->partials;
    a.red.counter = h->counter;
    a.red.expected = expected;
    a.red.rec = h->rec;
    a.red.h0sum = h->zero;
    a.red.dxdy = 0.0;
    launch_ingest(a, h->stream);
    h->nlaunch++;
  }
  CUDA_TRY(h, cudaGetLastError());
  CUDA_TRY(h, cudaMemcpyAsync(h->h0sum, h->rec + kRecSumEta, sizeof(double),
                              cudaMemcpyDeviceToDevice, h->stream));
  // static hzero halo, once; in P2P mode also the state-0 halos (later steps
  // deliver them with the boundary rows): NCCL exchange, device copies between
  // virtual slabs, or stores into the neighbours' halos plus a signal (P2P).
  const bool p2p = h->halo_mode == SW2D_HALO_P2P;
  if (h->virt) {
    int rc = virtual_halo(h, -1);
    if (rc) return rc;
    if (p2p && (rc = virtual_halo(h, 0))) return rc;
  } else if (h->multi && p2p) {
    int rc = p2p_halo_init(h);
    if (rc) return rc;
  } else if (h->multi) {
    int rc = nccl_halo(h, -1, h->stream);
    if (rc) return rc;
  }
  h->wcur = 0;
  if (h->p.variant == SW2D_VARIANT_PAPER) {
    for (Slab& s : h->slabs) {
      PaperArgs a = paper_args(h, s);
      a.wet_out = s.W[0];
      launch_paper_init(a, h->stream);
      h->nlaunch++;
    }
    CUDA_TRY(h, cudaGetLastError());
  }
  int bad = 0;
  // the verdict reaches the host by a kernel store into mapped host memory,
  // not a copy: a device-to-host DMA would queue behind another handle's
  // multi-GB download on the same copy engine (the e2e pipeline, §8)
  publish_word<<<1, 1, 0, h->stream>>>(h->bad, h->bad_host);
  h->nlaunch++;
  CUDA_TRY(h, cudaGetLastError());
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  bad = *(volatile int*)h->bad_host;
  h->cur = 0;
  h->steps = 0;
  h->pending.clear();
  h->state_set = false;
  if (bad) return fail(h, SW2D_EINVAL, "non-finite value in the input state");
  CUDA_TRY(h, cudaEventRecord(h->ev_ready, h->stream));
  h->state_set = true;
  return SW2D_OK;
}

int sw2d_step(sw2d* h, int64_t nsteps) {
  NvtxRange nvtx_("sw2d_step");
  ENTER(h);
  if (nsteps < 0) return fail(h, SW2D_EINVAL, "nsteps must be >= 0");
  if (!h->state_set) return fail(h, SW2D_ESTATE, "sw2d_step before sw2d_set_state");
  if (h->p.variant == SW2D_VARIANT_PAPER) {
    for (int64_t i = 0; i < nsteps; ++i) {
      for (Slab& s : h->slabs) {
        launch_paper_step(paper_args(h, s), h->stream);
        h->nlaunch += 3;
      }
      CUDA_TRY(h, cudaGetLastError());
      h->wcur = 1 - h->wcur;
      if (h->red_level) {
        int rc = reduce_into(h, h->hist + (size_t)(h->steps % h->hist_len) * kRecN);
        if (rc) return rc;
      }
      h->steps++;
    }
    return SW2D_OK;
  }
  if (h->pk) {  // small grids: the persistent cooperative kernel
    Slab& sl = h->slabs[0];
    while (nsteps > 0) {
      const int64_t chunk =
          std::min<int64_t>(nsteps, h->red_level ? kPersistRedChunk : (int64_t)1 << 30);
      PersistArgs a{};
      for (int b = 0; b < 2; ++b) {
        a.E[b] = sl.E[b];
        a.U[b] = sl.U[b];
        a.V[b] = sl.V[b];
      }
      a.H0 = sl.H0;
      a.pitch = h->pitch;
      a.jbase = sl.j0 + 1 - kHaloRows;
      a.nx = (int)h->p.nx;
      a.ny = (int)h->p.ny;
      a.shape = h->pshape;
      a.th = h->pth;
      a.ntx = h->pntx;
      a.nty = h->pnty;
      a.cur = h->cur;
      a.nsteps = (int)chunk;
      a.flags = h->pflags;
      a.flag_base = h->pbase;
      a.ring = h->pring;
      a.ring_plane = h->p.nx * h->p.ny;
      a.c = h->coef;
      a.part = h->ppart;
      if (h->red_level) {
        set_dstep<<<1, 1, 0, h->stream>>>(h->dstep, (unsigned long long)h->steps);
        h->nlaunch++;
      }
      int e = 0;
      {
        // persistent launches of all handles of this process on this device
        // run one after another: two of them side by side could each hold
        // part of the SMs while their resident CTAs wait on tiles that
        // cannot start
        std::lock_guard<std::mutex> lk(g_persist_mu);
        cudaEvent_t& last = g_persist_last[h->device & 63];
        if (!last) CUDA_TRY(h, cudaEventCreateWithFlags(&last, cudaEventDisableTiming));
        CUDA_TRY(h, cudaStreamWaitEvent(h->stream, last, 0));
        e = launch_persist(a, h->pk, h->red_level, h->stream);
        if (!e) CUDA_TRY(h, cudaEventRecord(last, h->stream));
      }
      if (e) return fail(h, SW2D_ECUDA, std::string("cooperative launch: ") +
                                            cudaGetErrorString((cudaError_t)e));
      h->nlaunch++;
      if (h->red_level) {
        launch_fold_steps(h->ppart, h->pntx * h->pnty * persist_shape_warps(h->pshape),
                          (int)chunk, h->hist, h->hist_len,
                          h->dstep, h->h0sum, (double)h->p.dx * (double)h->p.dy, h->stream);
        h->nlaunch++;
      }
      CUDA_TRY(h, cudaGetLastError());
      const int64_t blocks = (chunk + h->pk - 1) / h->pk;
      h->cur ^= (int)(blocks & 1);
      h->pbase += (unsigned)chunk;
      h->steps += chunk;
      nsteps -= chunk;
    }
    return SW2D_OK;
  }
  // Small problems are bound by launch latency: replay a CUDA graph of
  // kGraphPasses passes (same kernels and arguments, one graph per starting
  // buffer parity); per-step diagnostics find their history slot on the
  // device, so they replay too.
  const int spl0 = !h->launches2.empty() ? 2 : 1;
  // (the legacy and per-thread default streams cannot be captured)
  const bool capturable = h->stream != cudaStreamLegacy && h->stream != cudaStreamPerThread &&
                          h->stream != nullptr;
  const bool graphs = !h->multi && capturable && graphs_enabled();
  while (graphs && nsteps >= (int64_t)kGraphPasses * spl0) {
    cudaGraphExec_t& g = h->graph[h->cur];
    if (!g || h->graph_spl != spl0) {
      if (g) cudaGraphExecDestroy(g);
      g = nullptr;
      for (int b = 0; b < 2; ++b)
        if (h->graph[b] && h->graph_spl != spl0) {
          cudaGraphExecDestroy(h->graph[b]);
          h->graph[b] = nullptr;
        }
      h->graph_spl = spl0;
      const int cur0 = h->cur;
      const int64_t steps0 = h->steps, launches0 = h->nlaunch;
      cudaGraph_t graph = nullptr;
      CUDA_TRY(h, cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
      int rc = SW2D_OK;
      h->capturing = true;
      h->cap_step = 0;
      for (int i = 0; i < kGraphPasses && rc == SW2D_OK; ++i) rc = run_pass(h, spl0);
      h->capturing = false;
      if (rc == SW2D_OK && h->red_level && spl0 == 2 && h->kind == 2)
        launch_fold_steps(h->gpart, h->step_blocks2, kGraphPasses * spl0, h->hist, h->hist_len,
                          h->dstep, h->h0sum, (double)h->p.dx * (double)h->p.dy, h->stream);
      else if (rc == SW2D_OK && h->red_level)
        ring_scatter<<<1, 256, 0, h->stream>>>(h->grec, h->hist, h->hist_len, h->dstep,
                                               kGraphPasses * spl0);
      const cudaError_t ce = cudaStreamEndCapture(h->stream, &graph);
      h->cur = cur0;  // capture only recorded the passes
      h->steps = steps0;
      h->nlaunch = launches0;
      if (rc) return rc;
      CUDA_TRY(h, ce);
      const cudaError_t ie = cudaGraphInstantiate(&g, graph, 0);
      cudaGraphDestroy(graph);
      CUDA_TRY(h, ie);
    }
    if (h->red_level) {  // the graph's first step: its history slot base
      set_dstep<<<1, 1, 0, h->stream>>>(h->dstep, (unsigned long long)h->steps);
      h->nlaunch++;
    }
    CUDA_TRY(h, cudaGraphLaunch(g, h->stream));
    h->nlaunch += (int64_t)kGraphPasses * (int64_t)(h->launches2.empty() ? h->launches.size()
                                                                        : h->launches2.size()) +
                  (h->red_level ? 1 : 0);
    h->steps += (int64_t)kGraphPasses * spl0;
    nsteps -= (int64_t)kGraphPasses * spl0;  // kGraphPasses is even: parity unchanged
  }
  while (nsteps > 0) {
    const int spl = (nsteps >= 2 && !h->launches2.empty()) ? 2 : 1;
    int rc = run_pass(h, spl);
    if (rc) return rc;
    nsteps -= spl;
  }
  if (h->multi && !h->pending.empty()) {
    CUDA_TRY(h, cudaStreamWaitEvent(h->comm, h->ev_ready, 0));
    int rc = flush_pending(h);
    if (rc) return rc;
  }
  if (h->multi && h->red_level) {
    // later work on the compute stream (reads of the history) follows the allreduces
    CUDA_TRY(h, cudaEventRecord(h->ev_halo, h->comm));
    CUDA_TRY(h, cudaStreamWaitEvent(h->stream, h->ev_halo, 0));
  }
  return SW2D_OK;
}

int sw2d_run_snapshots(sw2d* h, int64_t nsteps, int64_t every, float* out_eta,
                       int64_t nsnap) {
  NvtxRange nvtx_("sw2d_run_snapshots");
  ENTER(h);
  if (!out_eta || every < 1 || nsteps < 0 || nsnap != nsteps / every)
    return fail(h, SW2D_EINVAL, "need every >= 1, nsnap == nsteps / every, out_eta");
  if (!h->state_set) return fail(h, SW2D_ESTATE, "sw2d_run_snapshots before sw2d_set_state");
  const int64_t nx = h->p.nx, hj0 = h->slabs.front().j0;
  int64_t rows = 0;
  for (Slab& s : h->slabs) rows += s.nrows;
  const size_t bytes = (size_t)rows * (size_t)nx * sizeof(float);
  if (bytes > h->snap_bytes) {
    for (int b = 0; b < 2; ++b) {
      cudaFree(h->snap[b]);
      h->snap[b] = nullptr;
    }
    h->snap_bytes = 0;
    for (int b = 0; b < 2; ++b) CUDA_TRY(h, cudaMalloc(&h->snap[b], bytes));
    h->snap_bytes = bytes;
  }
  if (!h->copy) {
    CUDA_TRY(h, cudaStreamCreateWithFlags(&h->copy, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_snap[b], cudaEventDisableTiming));
      CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_copied[b], cudaEventDisableTiming));
    }
  }
  const size_t wbytes = (size_t)nx * sizeof(float);
  const size_t dp = (size_t)h->pitch * sizeof(float);
  for (int64_t k = 0; k < nsnap; ++k) {
    int rc = sw2d_step(h, every);
    if (rc) return rc;
    const int b = (int)(k & 1);
    if (k >= 2) CUDA_TRY(h, cudaStreamWaitEvent(h->stream, h->ev_copied[b], 0));
    for (Slab& s : h->slabs)  // pack the interior of eta (device to device)
      CUDA_TRY(h, cudaMemcpy2DAsync(h->snap[b] + (size_t)(s.j0 - hj0) * (size_t)nx, wbytes,
                                    s.E[h->cur] + kHaloRows * h->pitch + 1 + kColOff, dp,
                                    wbytes, (size_t)s.nrows, cudaMemcpyDeviceToDevice,
                                    h->stream));
    CUDA_TRY(h, cudaEventRecord(h->ev_snap[b], h->stream));
    CUDA_TRY(h, cudaStreamWaitEvent(h->copy, h->ev_snap[b], 0));
    CUDA_TRY(h, cudaMemcpyAsync(out_eta + (size_t)k * (size_t)rows * (size_t)nx, h->snap[b],
                                bytes, cudaMemcpyDefault, h->copy));
    CUDA_TRY(h, cudaEventRecord(h->ev_copied[b], h->copy));
  }
  {
    int rc = sw2d_step(h, nsteps - nsnap * every);
    if (rc) return rc;
  }
  CUDA_TRY(h, cudaStreamSynchronize(h->copy));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  return SW2D_OK;
}

int sw2d_sync(sw2d* h) {
  ENTER(h);
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  if (h->comm) CUDA_TRY(h, cudaStreamSynchronize(h->comm));
  if (h->comm_nccl) {
    ncclResult_t ar = ncclSuccess;
    NCCL_TRY(h, sw2d_host::nccl().CommGetAsyncError(h->comm_nccl, &ar));
    NCCL_TRY(h, ar);
  }
  return SW2D_OK;
}

int sw2d_reduce(sw2d* h, int op, double* out) {
  NvtxRange nvtx_("sw2d_reduce");
  ENTER(h);
  if (!out || op < 0 || op >= SW2D_RED_N) return fail(h, SW2D_EINVAL, "bad op / out");
  if (!h->state_set) return fail(h, SW2D_ESTATE, "sw2d_reduce before sw2d_set_state");
  if (p2p_real(h)) {  // this rank's record in its exchange slot, combined on comm
    int rc = guard_slots(h, h->xseq, 1);
    if (!rc) rc = reduce_into(h, xslot(h->sync, h->nranks, h->xseq, h->rank));
    if (rc) return rc;
    CUDA_TRY(h, cudaEventRecord(h->ev_ready, h->stream));
    CUDA_TRY(h, cudaStreamWaitEvent(h->comm, h->ev_ready, 0));
    rc = p2p_exchange(h, h->xseq, 1, h->rec, nullptr);
    if (rc) return rc;
    h->xseq++;
    CUDA_TRY(h, cudaEventRecord(h->ev_halo, h->comm));
    CUDA_TRY(h, cudaStreamWaitEvent(h->stream, h->ev_halo, 0));
  } else {
    int rc = reduce_into(h, h->rec);
    if (rc) return rc;
    if (h->multi && (rc = nccl_allreduce_rec(h, h->rec, h->rec, h->stream))) return rc;
  }
  double rec[kRecN];
  CUDA_TRY(h, cudaMemcpyAsync(rec, h->rec, sizeof(rec), cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  *out = rec_value(rec, op);
  return SW2D_OK;
}

int sw2d_reduce_history(sw2d* h, int op, double* out, int64_t n) {
  NvtxRange nvtx_("sw2d_reduce_history");
  ENTER(h);
  if (!out || op < 0 || op >= SW2D_RED_N || n < 0)
    return fail(h, SW2D_EINVAL, "bad op / out / n");
  if (!(h->p.reduce_every_step & (1u << op)))
    return fail(h, SW2D_EINVAL, "op not in reduce_every_step");
  if (n > h->steps || n > h->hist_len)
    return fail(h, SW2D_EINVAL, "n exceeds the steps taken or history_len");
  if (n == 0) return SW2D_OK;
  std::vector<double> ring((size_t)h->hist_len * kRecN);
  CUDA_TRY(h, cudaMemcpyAsync(ring.data(), h->hist, ring.size() * sizeof(double),
                              cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  for (int64_t i = 0; i < n; ++i) {
    const int64_t step = h->steps - n + i;
    out[i] = rec_value(ring.data() + (size_t)(step % h->hist_len) * kRecN, op);
  }
  return SW2D_OK;
}

int sw2d_get_state(sw2d* h, float* eta, float* u, float* v, uint8_t* wet) {
  NvtxRange nvtx_("sw2d_get_state");
  ENTER(h);
  if (!h->state_set) return fail(h, SW2D_ESTATE, "sw2d_get_state before sw2d_set_state");
  const int64_t nx = h->p.nx, hj0 = h->slabs.front().j0;
  int64_t total_rows = 0;
  for (Slab& s : h->slabs) total_rows += s.nrows;
  if (wet) {
    const size_t need = (size_t)total_rows * (size_t)nx;
    if (need > h->wetbuf_bytes) {
      cudaFree(h->wetbuf);
      h->wetbuf = nullptr;
      h->wetbuf_bytes = 0;
      CUDA_TRY(h, cudaMalloc(&h->wetbuf, need));
      h->wetbuf_bytes = need;
    }
  }
  // device arrays: a device copy out of the pitched fields; host arrays: the
  // same into the dense stage, then one contiguous DMA per field
  float* outp[3] = {eta, u, v};
  float* dense[3] = {nullptr, nullptr, nullptr};
  const size_t cells = (size_t)total_rows * (size_t)nx;
  for (int f = 0; f < 3; ++f) {
    if (!outp[f]) continue;
    if (is_device_ptr(outp[f])) {
      dense[f] = outp[f];
      continue;
    }
    int rc = ensure_stage(h, 4, total_rows);
    if (rc) return rc;
    dense[f] = h->stage + (size_t)f * cells;
  }
  for (Slab& s : h->slabs) {
    const size_t off = (size_t)(s.j0 - hj0) * (size_t)nx;
    const float* src[3] = {s.E[h->cur], s.U[h->cur], s.V[h->cur]};
    for (int f = 0; f < 3; ++f)
      if (dense[f])
        launch_copy_rows(h, dense[f] + off, nx, src[f] + kHaloRows * h->pitch + 1 + kColOff,
                         h->pitch, s.nrows);
    if (wet) {
      launch_wet(s.E[h->cur], s.H0, h->pitch, s.nrows, (int)nx, h->p.hmin,
                 h->wetbuf + off, h->stream);
      h->nlaunch++;
    }
  }
  CUDA_TRY(h, cudaGetLastError());
  for (int f = 0; f < 3; ++f)
    if (dense[f] && dense[f] != outp[f])
      CUDA_TRY(h, cudaMemcpyAsync(outp[f], dense[f], cells * sizeof(float),
                                  cudaMemcpyDeviceToHost, h->stream));
  if (wet)
    CUDA_TRY(h, cudaMemcpyAsync(wet, h->wetbuf, (size_t)total_rows * (size_t)nx,
                                cudaMemcpyDefault, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  return SW2D_OK;
}

int64_t sw2d_launch_count(const sw2d* h) { return h ? h->nlaunch : -1; }

const char* sw2d_plan(const sw2d* h) { return h ? h->plan_text.c_str() : ""; }

void sw2d_destroy(sw2d* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  if (h->comm) cudaStreamSynchronize(h->comm);
  free_all(h);
  delete h;
}

const char* sw2d_strerror(int code) {
  switch (code) {
    case SW2D_OK: return "ok";
    case SW2D_EINVAL: return "invalid argument";
    case SW2D_ENOMEM: return "out of device memory";
    case SW2D_ECUDA: return "CUDA error";
    case SW2D_ENCCL: return "NCCL error";
    case SW2D_ESTATE: return "state not set";
    case SW2D_EUNSUPPORTED: return "unsupported";
    default: return "unknown status";
  }
}

const char* sw2d_last_error(const sw2d* h) {
  return h ? h->err.c_str() : t_create_err.c_str();
}

}  // extern "C"
