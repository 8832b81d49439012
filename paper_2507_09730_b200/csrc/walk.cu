// walk.cu -- the floating-random-walk engine on sm_100a (configs C3-C5).
//
// Reference semantics (relative to /root/reference/proj):
//   Engine::run_walk          src/engine.cpp:352-376   (walk driver)
//   Engine::first_transition  src/engine.cpp:201-288   (ladder + weight)
//   Engine::transition        src/engine.cpp:290-350   (snap, cached, MW)
//   sample_gaussian           src/engine.cpp:126-148
//   walk_lattice<LazyField>   src/microwalk.cpp:44-156 (lazy MicroWalk)
//   Structure queries         src/geometry.cpp:31-80, :357-396
//   profile_key / round_sig   src/sgf_cache.cpp:13-51
//   sample_panel              src/sgf.cpp:301-308
//
// B200 design: a wavefront engine over a resident pool of
// walk slots, so that the long MicroWalk step loops never share a warp with
// the (divergent, scan-heavy) geometry queries:
//   k_spawn    Gaussian sample + first-transition ladder for free slots
//   k_advance  snap / ground tests, free cube, stratification probe; cached
//              (stratified) hops are taken inline; a general cube is
//              compiled into a MicroWalk job (clipped dielectric boxes in
//              voxel-index space + the start node's cell) and queued
//   k_mw       persistent MicroWalk kernel: one hop per thread, threads
//              re-armed from the queue; steps inside a uniform cell use the
//              integer threshold compare of mw_grid.cu, steps next to an
//              interface use the reference's f64 scan with alphas read from
//              a palette-pair table (no division)
//   k_reduce*  per-walk records -> per-terminal tallies in a fixed order
// All geometry and voxel-centre arithmetic is compiled with -fmad=false so
// it rounds exactly like the reference (x86-64 baseline, no contraction).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "frw_internal.h"
#include "frw_rng.cuh"

namespace frw {
namespace {

constexpr int KMAX = 64;    // clipped boxes (conductors + dielectrics) per MicroWalk cube
constexpr int NMAX = 128;   // lattice size cap (layers per key; face distances stay < 128,
                            // the byte tricks of mw_step / mw_jump need that)
constexpr int PMAX = 40;    // palettes up to PMAX classes keep the alpha table in shared memory
                            // (12.8 KB; larger ones divide, the same IEEE quotient)
constexpr int kClassMax = 0x7FFF;  // distinct permittivities (15-bit class ids)
constexpr int kSlotsDefault = 1 << 20;
constexpr int kMwSlice = 64;   // MicroWalk super-steps per hop and k_mw visit
constexpr int kAdvSlice = 16;  // transitions per walk and k_advance visit
constexpr int kGridMinConductors = 24;  // conductor bins above this count
// Cell atlas of a MicroWalk job (u64 words per slot).  Along each axis the
// clipped boxes' faces cut [0, n) into segments; bm[a] holds one bit per
// segment start.  mask[a][s] is the set of clipped boxes (bit q = box q)
// spanning segment s, so the boxes containing a cell are the AND of its
// three segment masks and its class is a bit scan.  FDM jobs (n <= 32) keep
// every bitmap in one word.
constexpr int kAtMask = 0;    // [3][64] segment masks
constexpr int kAtBm = 192;    // [3] segment-start bitmaps
constexpr int kAtCls = 195;   // [KMAX] u16 palette class of each clipped dielectric box
constexpr int kAtlasWords = 211;
constexpr double kEps0 = 8.8541878128e-12;  // constants.hpp:5
constexpr double kMPerNm = 1e-9;            // constants.hpp:6



// Device bounds checks (compute-sanitizer is unavailable on the GPU pool):
// a build with -DFRW_DEBUG_CHECKS tests every queue push and pop, slot and
// job index, walk record index, lattice node and table index below; the
// first failure records its source line and fails the call (FRW_ECUDA,
// "device check failed at walk.cu:LINE").  Compiled out by default.
#ifdef FRW_DEBUG_CHECKS
#define FRW_DCHECK(C, cond)                                                               \
  do {                                                                                    \
    if (!(cond)) {                                                                        \
      atomicCAS(&(C)->chk_line, 0ull, static_cast<unsigned long long>(__LINE__));         \
      atomicCAS(&(C)->err, 0ull, static_cast<unsigned long long>(-FRW_ECUDA));                                                            \
    }                                                                                     \
  } while (0)
#else
#define FRW_DCHECK(C, cond) static_cast<void>(0)
#endif

// Phase clocks (experiment builds, -DFRW_PHASE_CLOCKS): clock64 spans of the
// walk kernels' phases summed per phase (g_ph[i]) with event counts
// (g_ph[16 + i]); frw_run_walks prints them to stderr after the call.
#ifdef FRW_PHASE_CLOCKS
__device__ unsigned long long g_ph[256 * 32];  // 256 rows (spread by thread): no hot address
#define PH_ROW (((blockIdx.x * blockDim.x + threadIdx.x) & 255) * 32)
// completion times of the walks k_tail finishes, 0.25 ms buckets from the
// launch (g_tail_t0: globaltimer of the launch's first lane)
__device__ unsigned long long g_tail_hist[256];
__device__ unsigned long long g_tail_t0;
__device__ int g_in_tail;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PH_T0(v) const long long v = clock64()
#define PH_ADD(i, v)                                                              \
  do {                                                                            \
    atomicAdd(&g_ph[PH_ROW + (i)], static_cast<unsigned long long>(clock64() - (v))); \
    atomicAdd(&g_ph[PH_ROW + 16 + (i)], 1ull);                                    \
  } while (0)
#else
#define PH_T0(v) static_cast<void>(0)
#define PH_ADD(i, v) static_cast<void>(0)
#endif

enum : uint8_t { S_FREE = 0, S_ACTIVE = 1, S_NEED_MW = 2, S_PARKED = 3, S_MW_CARRY = 4 };


// ---------------------------------------------------------------------------
// device-side views

// Uniform bin grid over the world box with per-bin conductor lists (CSR),
// used by the conductor queries once a structure has many conductors.  A
// box is listed in every bin its closed extent overlaps, with bins taken by
// floor((x - lo) / bs) on host and device alike (monotone, identical
// rounding), so every query below returns exactly the linear scan's result.
struct DGrid {
  int dims[3];          // 0: no grid, linear scans
  double lo[3], bs[3], ibs[3];  // origin, bin size per axis, its inverse
  double bsmin;
  const int* cstart;    // [bins + 1] conductors overlapping the bin (CSR)
  const int* citem;
  const int* nstart;    // [bins + 1] conductors that can be nearest to a
  const int* nitem;     //   point of the bin (see frw_upload_structure)
  const int* dstart;    // [bins + 1] small dielectrics overlapping the bin
  const int* ditem;
  const int* dlarge;    // dielectrics spanning many bins: always candidates
  int ndlarge;
};

struct DStruct {
  int nc, nd, P, bg;
  const double* cbox;   // [nc][6]
  const double* dbox;   // [nd][6]
  const uint16_t* dcls; // [nd] palette class
  const double* pal;    // [P]
  const double* alpha;  // [P][P] when P <= PMAX: alpha[nb*P + self] = e_nb/(e_nb+e_self)
  const double* rpal;   // [P] value rounded to 6 significant digits
  double world[6];
  DGrid g;
};

struct DSgf {
  int cap;                   // power of two
  const uint64_t* hash;      // [cap]
  const int* entry;          // [cap], -1 empty
  const int* axis;           // [entries]
  const double* keys;        // [entries][NMAX]
  const double* pitch;       // [entries]
  const double* const* data; // [entries] -> cdf[P], probs[P], kern[3][P]
  const int* uentry;         // [P] entry of the uniform key of each palette class, -1
};

// Lattice jumps (Philox mode only).  Inside one cell every alpha is 1/2, so
// the MicroWalk is the simple symmetric walk there.  From a node whose six
// face distances are all >= m the walk's first hit of the L-inf sphere of
// radius m is the discrete harmonic measure of the (2m-1)^3 interior: the
// surface Green's function of the uniform cube with n' = 2m-1 nodes (the
// device solve of sgf_solve.cu).  By the strong Markov property replacing
// those steps by one draw from it leaves the law of the hop's exit (and the
// expected step count) unchanged.  Per radius m: the face law over the
// (2m-1)^2 positions of a face (face chosen uniformly: the cube is
// octahedrally symmetric) as a Walker alias table -- u64 acceptance
// thresholds and u16 aliases, one lookup and no scan -- and E[tau] in 32.32
// fixed point.  The kernels stage the tables of the radii that fit
// (kJumpSm entries, all of them for n <= 24) in shared memory.
struct JumpMeta {
  uint32_t off;        // into DJump::prob / alias
  uint32_t K;          // side^2 positions
  uint32_t magic;      // ceil(2^32 / side): idx / side = umulhi(idx, magic)
  uint32_t side;       // 2m - 1
  uint64_t esteps;     // E[tau] * 2^32
};
constexpr int kJumpMetaMax = 32;   // radii 0..31
constexpr int kJumpSm = 2048;      // alias entries staged in shared memory
struct DJump {
  int mmax;  // largest radius tabulated; < 2: jumps off
  int twice; // a second jump from words 2-3 of the block when it fits
  int hom;   // jumps across homogeneous balls beyond the walker's cell (mw_hom_radius)
  int msm;   // radii <= msm read prob_s / alias_s (shared memory)
  const JumpMeta* meta;   // [mmax + 1]
  const uint64_t* prob;   // per radius: K acceptance thresholds (u64 fractions)
  const uint16_t* alias;  // per radius: K aliases
  const uint64_t* prob_s; // shared-memory copies of the first radii's tables
  const uint16_t* alias_s;
};
struct JumpSmem {
  JumpMeta meta[kJumpMetaMax];
  uint64_t prob[kJumpSm];
  uint16_t alias[kJumpSm];
};

struct DParams {
  DJump jump;
  int n, panels, mode, rng;
  double snap;
  double expansion;
  long long hop_cap;
  uint64_t seed, mixed_seed;
  double gbox[6], fcdf[6], area;
  uint64_t walk_begin;
  long long count;
  int master;
  // time slices of the wavefront rounds (0: unlimited): super-steps of one
  // MicroWalk hop per k_mw visit, transitions of one walk per k_advance visit
  int mw_slice, adv_slice;
  // k_flow: SM pairs (of flow_sms) that run transitions; the others run MicroWalk hops
  int flow_adv, flow_sms;
};

struct WalkRec {  // per walk id, written once when the walk terminates
  double weight;
  uint64_t mw_steps;
  int slot;
  uint32_t cached;
  uint32_t mw;
  uint8_t aborted, branch, resampled, done;
};

struct DSlots {
  int S;
  int J;                 // job entries (slot capacity + tail lanes)
  long long count;       // walk records of the call (FRW_DEBUG_CHECKS)
  int jtail;             // first job entry of the k_tail lanes (one per lane,
                         // after the capacity's slots: compiled, walked and
                         // re-compiled by the same lane, so they stay in L2)
  uint8_t* state;
  long long* wid;        // walk index relative to walk_begin
  double* p;             // [S][3]
  double* weight;
  uint64_t* rng;         // SplitMix64 state or Philox block counter
  int* hops;
  uint32_t* cached;
  uint32_t* mw;
  uint64_t* mwsteps;
  uint8_t* branch;
  uint8_t* resampled;
  // MicroWalk job compiled by k_advance
  double* cube;          // [S][4] center, half width
  uint16_t* nbox;        // [J] conductor boxes among the clipped boxes | boxes << 8
  uint64_t* boxes;       // [S][KMAX] lo.xyz, hi.xyz, class / conductor index
  uint64_t* atlas;       // [S][kAtlasWords] cell atlas of an FDM job (build_atlas; k_fdm)
  uint8_t* mwkind;       // [S] 0 plain MicroWalk job, 1 expanded (MicroWalk-E), 2 FDM
  // a MicroWalk hop carried to the next round (S_MW_CARRY): node, steps so far
  uint32_t* mwnode;
  int* mwhsteps;
  uint64_t* mwhj;        // its homogeneous-radius bound: hom | (hq + 1) << 8 | hnode << 32
};

// Work queues of one round: k_spawn and the previous round's k_mw fill the
// ACTIVE queue; k_advance drains it (one transition per pop, lanes re-armed
// as their walk leaves the stage) and fills the MicroWalk queue; k_mw drains
// that and fills the next round's ACTIVE queue.
struct DCounters {
  unsigned long long next;       // next new walk id
  unsigned long long done;       // walks finished
  unsigned long long qlen;       // MicroWalk queue length
  unsigned long long qhead;      // MicroWalk queue head
  unsigned long long alen;       // ACTIVE queue length (this round)
  unsigned long long ahead;      // ACTIVE queue head
  unsigned long long a2len;      // ACTIVE queue of the next round
  unsigned long long nmiss;      // miss records written
  unsigned long long npend;      // pending restarts available
  unsigned long long pend_head;  // pending restarts consumed
  unsigned long long nretry;     // walks parked by a miss this round
  unsigned long long err;        // error code (first)
  unsigned long long gen_steps;  // MicroWalk steps next to a cell face
  unsigned long long cell_chg;   // MicroWalk moves into another cell
  unsigned long long npark;      // walks parked mid-walk (their slots kept)
  // k_flow: ring heads/tails (ACTIVE, MicroWalk) and walks still in the flow
  unsigned long long fah, fat, fmh, fmt, flive;
  unsigned long long jumps;      // MicroWalk lattice jumps (Philox mode)
  unsigned long long jsteps;     // lattice steps the jumps stand for (their E[tau])
  unsigned long long q2len;      // MicroWalk queue of the next round (carried hops)
  unsigned long long dqlen, dqhead;  // dense MicroWalk hops of this round (k_mw_dense)
  unsigned long long cqlen;          // walks queued for k_compile this round
  unsigned long long dense_hops;     // dense hops run (all rounds)
  // k_tail: warp cycles in MicroWalk super-steps / in the whole loop, for
  // the MicroWalk share of the tail's device time (T_MW, engine.cpp:322-345)
  unsigned long long tail_mw_cyc, tail_all_cyc;
  unsigned long long chk_line;   // FRW_DEBUG_CHECKS: line of the first failed device check
};

constexpr int kMissMax = 4096;
constexpr uint8_t kDense = 4, kDenseCond = 8;  // mwkind flags of a dense hop (k_mw_dense)
struct DMiss {
  int* axis;        // [kMissMax]
  double* layers;   // [kMissMax][NMAX]
  long long* retry; // [2S] walk ids whose first transition missed (restart)
  long long* pend;  // [2S] walk ids to restart
  int* park;        // [2S] slots of walks parked mid-walk by a miss (resume)
  int* dense;       // [S] slots whose MicroWalk hop needs the dense grid (k_mw_dense)
  long long cap;    // slot capacity (retry/pend/park hold 2 cap)
};

// ---------------------------------------------------------------------------
// exact reference arithmetic helpers (std::max / std::min semantics)

__device__ __forceinline__ double mx(double a, double b) { return a < b ? b : a; }
__device__ __forceinline__ double mn(double a, double b) { return b < a ? b : a; }

// Box::chebyshev_to (geometry.cpp:31-37)
__device__ __forceinline__ double cheb_to(const double* b, const double p[3]) {
  double d = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a) d = mx(d, mx(__ldg(b + a) - p[a], p[a] - __ldg(b + 3 + a)));
  return mx(d, 0.0);
}
// Box::chebyshev_to_wall (geometry.cpp:39-45)
__device__ __forceinline__ double cheb_wall(const double* b, const double p[3]) {
  double d = INFINITY;
#pragma unroll
  for (int a = 0; a < 3; ++a) d = mn(d, mn(p[a] - b[a], b[3 + a] - p[a]));
  return d;
}
// Box::contains (geometry.hpp:37-40); `b` may live in any address space
// (short-circuit on purpose: the long scans of permittivity_at -- dense hop
// grids classify every voxel centre -- mostly stop at the first compare; a
// branch-free six-load version cost C5 a third of its large-call throughput)
__device__ __forceinline__ bool box_contains(const double* b, const double p[3]) {
  return p[0] >= b[0] && p[0] <= b[3] && p[1] >= b[1] && p[1] <= b[4] && p[2] >= b[2] &&
         p[2] <= b[5];
}

// Structure::conductor_at (geometry.cpp:57-62): declaration index or -1
__device__ __forceinline__ int bin_of(const DGrid& g, int a, double x) {
  const int i = static_cast<int>(floor((x - g.lo[a]) * g.ibs[a]));
  return min(max(i, 0), g.dims[a] - 1);
}

// first declared conductor within Chebyshev distance tol of p, -1 if none:
// its box overlaps the bins of [p - tol, p + tol]
__device__ int grid_conductor_within(const DStruct& s, const double p[3], double tol) {
  const DGrid& g = s.g;
  int b0[3], b1[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    b0[a] = bin_of(g, a, p[a] - tol);
    b1[a] = bin_of(g, a, p[a] + tol);
  }
  int best = 0x7FFFFFFF;
  // (rolled loops: one copy of the distance test -- the walk kernels are
  // instruction-fetch bound)
#pragma unroll 1
  for (int z = b0[2]; z <= b1[2]; ++z)
#pragma unroll 1
    for (int y = b0[1]; y <= b1[1]; ++y)
#pragma unroll 1
      for (int x = b0[0]; x <= b1[0]; ++x) {
        const int bin = (z * g.dims[1] + y) * g.dims[0] + x;
#pragma unroll 1
        for (int q = __ldg(g.cstart + bin), e = __ldg(g.cstart + bin + 1); q < e; ++q) {
          const int c = __ldg(g.citem + q);
          if (c < best && cheb_to(s.cbox + 6 * c, p) <= tol) best = c;
        }
      }
  return best == 0x7FFFFFFF ? -1 : best;
}

// min(r, Chebyshev distance from p to every conductor) over the bin's
// nearest-candidate list, which holds every conductor that can be closest to
// some point of the bin (or closer than the world wall there), so the
// minimum equals the linear scan's.  *inside: some conductor contains p
// (such a conductor is a candidate of p's bin: its distance there is 0).
__device__ double grid_min_cheb(const DStruct& s, const double p[3], double r, bool* inside) {
  const DGrid& g = s.g;
  const int bin = (bin_of(g, 2, p[2]) * g.dims[1] + bin_of(g, 1, p[1])) * g.dims[0] +
                  bin_of(g, 0, p[0]);
#pragma unroll 1
  for (int q = __ldg(g.nstart + bin), e = __ldg(g.nstart + bin + 1); q < e; ++q) {
    const double d = cheb_to(s.cbox + 6 * __ldg(g.nitem + q), p);
    if (d <= 0) *inside = true;
    if (d <= r) r = d;
  }
  return r;
}

// Candidates for "every box of a kind meeting the closed region [lo, hi]",
// ascending declaration order, deduplicated: the boxes listed in the bins the
// region overlaps (plus, for dielectrics, the large ones).  Returns -1 when
// there is no grid, the region spans too many bins or the list overflows:
// the caller then scans every box, so results never depend on the bins.
constexpr int kCandMax = 96;
constexpr int kCandBins = 64;
__device__ __forceinline__ bool cand_insert(int* a, int& n, int v) {
  int i = n;
  while (i > 0 && a[i - 1] > v) --i;
  if (i > 0 && a[i - 1] == v) return true;
  if (n == kCandMax) return false;
  for (int j = n; j > i; --j) a[j] = a[j - 1];
  a[i] = v;
  ++n;
  return true;
}
__device__ int grid_candidates(const DStruct& s, bool diel, const double* cb, int* out) {
  const DGrid& g = s.g;
  if (!g.dims[0]) return -1;
  int b0[3], b1[3], nb = 1;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    b0[a] = bin_of(g, a, cb[a]);
    b1[a] = bin_of(g, a, cb[3 + a]);
    nb *= b1[a] - b0[a] + 1;
  }
  if (nb > kCandBins) return -1;
  const int* st = diel ? g.dstart : g.cstart;
  const int* it = diel ? g.ditem : g.citem;
  int n = 0;
  if (diel)
    for (int q = 0; q < g.ndlarge; ++q)
      if (!cand_insert(out, n, __ldg(g.dlarge + q))) return -1;
  for (int z = b0[2]; z <= b1[2]; ++z)
    for (int y = b0[1]; y <= b1[1]; ++y)
      for (int x = b0[0]; x <= b1[0]; ++x) {
        const int bin = (z * g.dims[1] + y) * g.dims[0] + x;
        for (int q = __ldg(st + bin), e = __ldg(st + bin + 1); q < e; ++q)
          if (!cand_insert(out, n, __ldg(it + q))) return -1;
      }
  return n;
}

__device__ int conductor_at(const DStruct& s, const double p[3], double tol) {
  if (s.g.dims[0]) return grid_conductor_within(s, p, tol);
  for (int c = 0; c < s.nc; ++c)
    if (cheb_to(s.cbox + 6 * c, p) <= tol) return c;
  return -1;
}

// Structure::max_free_cube (geometry.cpp:64-80); false when the reference
// would throw (point outside the world or inside a conductor)
__device__ bool max_free_cube(const DStruct& s, const double p[3], double* h) {
  double r = cheb_wall(s.world, p);
  if (r <= 0) return false;
  if (s.g.dims[0]) {
    bool inside = false;
    r = grid_min_cheb(s, p, r, &inside);
    if (inside) return false;
    *h = r;
    return true;
  }
  for (int c = 0; c < s.nc; ++c) {
    const double d = cheb_to(s.cbox + 6 * c, p);
    if (d <= 0) return false;
    if (d <= r) r = d;
  }
  *h = r;
  return true;
}

// The geometry prologue of Engine::transition (engine.cpp:293-298) in one
// pass over the conductors: conductor_at(p, snap) -> its declaration index;
// the world wall within snap -> -1 (ground); else the max free cube half
// width in *h and -3.  (A conductor at d <= 0 would have been caught by the
// snap test first, so max_free_cube's inside-conductor throw cannot fire.)
__device__ int hop_scan(const DStruct& s, const double p[3], double snap, double* h) {
  const double wall = cheb_wall(s.world, p);
  if (s.g.dims[0]) {
    const int c = grid_conductor_within(s, p, snap);
    if (c >= 0) return c;
    if (wall <= snap) return -1;
    bool inside = false;
    const double r = grid_min_cheb(s, p, wall, &inside);
    if (r <= 0) return -2;
    *h = r;
    return -3;
  }
  double r = wall;
#pragma unroll 1
  for (int c = 0; c < s.nc; ++c) {
    const double d = cheb_to(s.cbox + 6 * c, p);
    if (d <= snap) return c;
    if (d <= r) r = d;
  }
  if (wall <= snap) return -1;
  if (r <= 0) return -2;
  *h = r;
  return -3;
}

// Structure::permittivity_at (geometry.cpp:47-55) as a palette class;
// -1 outside the world
__device__ int eps_class_at(const DStruct& s, const double p[3]) {
  if (!box_contains(s.world, p)) return -1;
  if (s.g.dims[0]) {  // the last declared box containing p: max index among candidates
    const DGrid& g = s.g;
    int best = -1;
#pragma unroll 1
    for (int q = 0; q < g.ndlarge; ++q) {
      const int d = __ldg(g.dlarge + q);
      if (d > best && box_contains(s.dbox + 6 * d, p)) best = d;
    }
    const int bin = (bin_of(g, 2, p[2]) * g.dims[1] + bin_of(g, 1, p[1])) * g.dims[0] +
                    bin_of(g, 0, p[0]);
#pragma unroll 1
    for (int q = __ldg(g.dstart + bin), e = __ldg(g.dstart + bin + 1); q < e; ++q) {
      const int d = __ldg(g.ditem + q);
      if (d > best && box_contains(s.dbox + 6 * d, p)) best = d;
    }
    return best < 0 ? s.bg : __ldg(s.dcls + best);
  }
  int cls = s.bg;
#pragma unroll 1
  for (int d = 0; d < s.nd; ++d)
    if (box_contains(s.dbox + 6 * d, p)) cls = __ldg(s.dcls + d);
  return cls;
}

// transit_cube (microwalk.hpp:39-44)
__device__ __forceinline__ void transit_cube(const double p[3], double hw, int n, double c[3],
                                             double* h) {
  if (n % 2 == 1) {
    c[0] = p[0];
    c[1] = p[1];
    c[2] = p[2];
    *h = hw;
    return;
  }
  const double delta = hw / (n + 1);
  *h = (hw - delta) * (1.0 - 1e-12);
  c[0] = p[0] + delta;
  c[1] = p[1] + delta;
  c[2] = p[2] + delta;
}

// surface_panel_center (sgf.cpp:38-49)
__device__ void panel_center(const double c[3], double h, int n, int panel, double out[3]) {
  const int face = panel / (n * n);
  const int rem = panel - face * n * n;
  const int u = rem % n, v = rem / n;
  const int axis = face >> 1;
  const double pitch = 2.0 * h / n;
  out[axis] = c[axis] + ((face & 1) ? 1 : -1) * h;
  const int b1 = axis == 0 ? 1 : 0;
  const int b2 = axis == 2 ? 1 : 2;
  out[b1] = c[b1] - h + (u + 0.5) * pitch;
  out[b2] = c[b2] - h + (v + 0.5) * pitch;
}

// geometry.cpp:15-19
__device__ __forceinline__ bool eps_equal(double a, double b) {
  return fabs(a - b) <= 1e-9 * mx(fabs(a), fabs(b));
}

// round_sig (sgf_cache.cpp:13-18).  Palette values use host-rounded copies;
// this device version serves the slice means of ladder branches 2-3.  The
// power of ten comes from exactly rounded literals, so it matches glibc
// except when |x| lies within ~1e-15 of a power of ten.
__device__ double round_sig6(double x) {
  if (x == 0 || !isfinite(x)) return x;
  const double e10 = floor(log10(fabs(x)));
  const int k = 5 - static_cast<int>(e10);
  double mag;
  if (k >= 0 && k <= 22) {
    mag = 1.0;
    for (int i = 0; i < k; ++i) mag *= 10.0;  // exact up to 1e22
  } else if (k < 0 && k >= -22) {
    const double neg[23] = {1e0,   1e-1,  1e-2,  1e-3,  1e-4,  1e-5,  1e-6,  1e-7,
                            1e-8,  1e-9,  1e-10, 1e-11, 1e-12, 1e-13, 1e-14, 1e-15,
                            1e-16, 1e-17, 1e-18, 1e-19, 1e-20, 1e-21, 1e-22};
    mag = neg[-k];
  } else {
    mag = pow(10.0, static_cast<double>(k));
  }
  return round(x * mag) / mag;
}

// ---------------------------------------------------------------------------
// random streams: one per walk

struct Rng {
  uint64_t s;  // parity: SplitMix64 state; philox: block counter
};

__device__ __forceinline__ uint64_t philox53(const DParams& P, uint64_t wid, uint32_t blk,
                                             uint32_t dom) {
  const uint64_t id = P.walk_begin + wid;
  const U32x4 o = philox4x32_10(
      {static_cast<uint32_t>(id), static_cast<uint32_t>(id >> 32), blk, dom},
      static_cast<uint32_t>(P.seed), static_cast<uint32_t>(P.seed >> 32));
  return (static_cast<uint64_t>(o.x) << 21) | (o.y >> 11);
}

// one 53-bit uniform integer (rng.hpp:25 in parity mode)
__device__ __forceinline__ uint64_t draw53(const DParams& P, long long wid, Rng& r) {
  if (P.rng == FRW_RNG_SPLITMIX_PARITY) return sm64_next(r.s) >> 11;
  return philox53(P, static_cast<uint64_t>(wid), static_cast<uint32_t>(r.s++), 0u);
}
__device__ __forceinline__ double uniform(const DParams& P, long long wid, Rng& r) {
  return static_cast<double>(draw53(P, wid, r)) * 0x1.0p-53;
}

// ---------------------------------------------------------------------------
// stratification probe + profile key (geometry.cpp:357-396, sgf_cache.cpp:29-51)

// returns the key axis (0..2) and rounded layers, or -1 (general cube),
// -2 (error: slice centre outside the world)
__device__ void clip_axis(double c, double h, int n, double lo, double hi, int* il, int* ih);
__device__ void clip_axis(double c, double h, double p, double ip, int n, double lo, double hi,
                          int* il, int* ih);

// The stratification probe of a transition cube, held in registers (no
// per-slice arrays: the walk kernels keep no local memory on this path).
// stratified_profile (geometry.cpp:357-396): the dielectric boxes meeting
// the OPEN cube; the first axis whose cross-section every one of them
// covers; the permittivity of slice t is that of the last-declared box whose
// closed extent contains the slice centre c - h + (t + 0.5) pitch along the
// axis (permittivity_at, geometry.cpp:47-55), else the background.  Along
// the axis each box covers an interval of slices (clip_axis), so the profile
// is a few (class, slice-bitmask) pairs: painting box q (in declaration
// order) clears its slices from every pair and adds them to its class's
// pair.  Structures whose stratified cubes meet more than kProfHits boxes or
// kProfCls classes fall back to classifying slice centres one by one.
constexpr int kProfHits = 6;
constexpr int kProfCls = 4;
struct Prof {
  int axis;      // key axis (profile_key: uniform profiles -> 0); -1 general cube, -2 error
  int raxis;     // the probe's axis (slice centres lie along it)
  int ucls;      // >= 0: every slice has this palette class
  int ovf;       // 1: slices classified one by one (eps_class_at)
  int cls[kProfCls];
  uint64_t msk[kProfCls];
};

__device__ __forceinline__ uint64_t slice_bits(int lo, int hi) {  // bits lo..hi (lo <= hi < 64)
  return (hi >= 63 ? ~0ull : (2ull << hi) - 1) & ~((1ull << lo) - 1);
}

// palette class of slice t
__device__ __forceinline__ int prof_class(const DStruct& s, const Prof& P, const double c[3],
                                          double h, int n, int t) {
  if (P.ucls >= 0) return P.ucls;
  if (!P.ovf) {
    int k = s.bg;
#pragma unroll
    for (int e = 0; e < kProfCls; ++e)
      if ((P.msk[e] >> t) & 1) k = P.cls[e];
    return k;
  }
  double p[3] = {c[0], c[1], c[2]};
  p[P.raxis] = c[P.raxis] - h + (t + 0.5) * (2.0 * h / n);
  return eps_class_at(s, p);
}

// the key's layer t: round_sig(layer, 6) (sgf_cache.cpp:29-51; host-rounded palette)
__device__ __forceinline__ double prof_layer(const DStruct& s, const Prof& P, const double c[3],
                                             double h, int n, int t) {
  return __ldg(s.rpal + prof_class(s, P, c, h, n, t));
}

// visits the dielectric boxes that can meet the closed region cb: the bins it
// overlaps plus the large boxes (duplicates possible), or every box
template <class F>
__device__ __forceinline__ void for_dielectrics_near(const DStruct& s, const double cb[6], F f) {
  const DGrid& g = s.g;
  if (g.dims[0]) {
    int b0[3], b1[3], nb = 1;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      b0[a] = bin_of(g, a, cb[a]);
      b1[a] = bin_of(g, a, cb[3 + a]);
      nb *= b1[a] - b0[a] + 1;
    }
    if (nb <= kCandBins) {
#pragma unroll 1
      for (int q = 0; q < g.ndlarge; ++q)
        if (!f(__ldg(g.dlarge + q))) return;
#pragma unroll 1
      for (int z = b0[2]; z <= b1[2]; ++z)
#pragma unroll 1
        for (int y = b0[1]; y <= b1[1]; ++y)
#pragma unroll 1
          for (int x = b0[0]; x <= b1[0]; ++x) {
            const int bin = (z * g.dims[1] + y) * g.dims[0] + x;
#pragma unroll 1
            for (int q = __ldg(g.dstart + bin), e = __ldg(g.dstart + bin + 1); q < e; ++q)
              if (!f(__ldg(g.ditem + q))) return;
          }
      return;
    }
  }
#pragma unroll 1
  for (int d = 0; d < s.nd; ++d)
    if (!f(d)) return;
}

// scls (optional): the palette class of every slice when the probe classifies
// slice centres one by one (P.ovf), so lookups need no second classification
__device__ Prof strat_probe(const DStruct& s, const double c[3], double h, int n,
                            uint16_t* scls = nullptr) {
  Prof P;
  P.axis = -1;
  P.raxis = 0;
  P.ucls = -1;
  P.ovf = 0;
#pragma unroll
  for (int e = 0; e < kProfCls; ++e) {
    P.cls[e] = -1;
    P.msk[e] = 0;
  }
  const double cb[6] = {c[0] - h, c[1] - h, c[2] - h, c[0] + h, c[1] + h, c[2] + h};
  // pass 1: the boxes meeting the open cube, their coverage, and up to
  // kProfHits of them in ascending declaration order (no duplicates)
  int hit[kProfHits];
#pragma unroll
  for (int i = 0; i < kProfHits; ++i) hit[i] = 0x7FFFFFFF;
  int nh = 0;
  bool cov0 = true, cov1 = true, cov2 = true, many = false;
  for_dielectrics_near(s, cb, [&](int d) {
    const double* b = s.dbox + 6 * d;
    double bb[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) bb[q] = __ldg(b + q);
    // Box::intersects_open (geometry.hpp:49-52), without short-circuit branches
    if (!((bb[0] < cb[3]) & (cb[0] < bb[3]) & (bb[1] < cb[4]) & (cb[1] < bb[4]) &
          (bb[2] < cb[5]) & (cb[2] < bb[5])))
      return true;
    // covers the cross-section perpendicular to axis a (geometry.cpp:372-380)
    const bool fx = bb[0] <= cb[0] && bb[3] >= cb[3], fy = bb[1] <= cb[1] && bb[4] >= cb[4],
               fz = bb[2] <= cb[2] && bb[5] >= cb[5];
    cov0 &= fy && fz;
    cov1 &= fx && fz;
    cov2 &= fx && fy;
    if (!(cov0 || cov1 || cov2)) return false;  // a general cube: stop scanning
    bool dup = false;
#pragma unroll
    for (int i = 0; i < kProfHits; ++i) dup |= hit[i] == d;
    if (!dup) {
      ++nh;
      int x = d;  // sorted insert (unrolled min/max bubble: stays in registers)
#pragma unroll
      for (int i = 0; i < kProfHits; ++i) {
        const int lo = min(hit[i], x), hi = max(hit[i], x);
        hit[i] = lo;
        x = hi;
      }
      many |= x != 0x7FFFFFFF;
    }
    return true;
  });
  // (the scan stops at the first box that breaks every axis' coverage,
  // before counting it: test coverage first)
  if (!(cov0 || cov1 || cov2)) return P;  // general cube
  if (nh == 0) {  // background only (geometry.cpp:367-368)
    P.axis = 0;
    P.ucls = s.bg;
    return P;
  }
  P.raxis = cov0 ? 0 : (cov1 ? 1 : 2);
  const int ax = P.raxis;
  // (the (class, slice-mask) pairs hold 64 slices: larger lattices classify
  // slice centres one by one)
  if (!many && n <= 64) {
    // pass 2: paint the hits' slice intervals in declaration order
    P.cls[0] = s.bg;
    P.msk[0] = n >= 64 ? ~0ull : (1ull << n) - 1;
    const double pitch = 2.0 * h / n, ipitch = 1.0 / pitch;
    // one rolled copy of the paint step: the hits leave the front of the
    // sorted register list one by one (static indices, no local memory)
#pragma unroll 1
    for (int i = 0; i < nh; ++i) {
      const int d = hit[0];
#pragma unroll
      for (int j = 0; j + 1 < kProfHits; ++j) hit[j] = hit[j + 1];
      int lo, hi;
      clip_axis(c[ax], h, pitch, ipitch, n, __ldg(s.dbox + 6 * d + ax),
                __ldg(s.dbox + 6 * d + 3 + ax), &lo, &hi);
      if (lo > hi) continue;
      const uint64_t m = slice_bits(lo, hi);
      const int k = __ldg(s.dcls + d);
      bool placed = false;
#pragma unroll
      for (int e = 0; e < kProfCls; ++e) {
        P.msk[e] &= ~m;
        if (P.cls[e] == k) {
          P.msk[e] |= m;
          placed = true;
        }
      }
      if (!placed) {  // a new class takes the first free pair
        bool put = false;
#pragma unroll
        for (int e = 0; e < kProfCls; ++e)
          if (!put && P.msk[e] == 0) {
            P.cls[e] = k;
            P.msk[e] = m;
            put = true;
          }
        if (!put) P.ovf = 1;
      }
    }
  } else {
    P.ovf = 1;
  }
  // uniform?  (StratifiedProfile::uniform compares raw permittivities with
  // eps_equal, geometry.cpp:351-355; profile_key normalises equal rounded
  // layers to axis 0, sgf_cache.cpp:40-42)
  if (!P.ovf) {
    int k0 = s.bg, present = 0, only = -1;
#pragma unroll
    for (int e = 0; e < kProfCls; ++e)
      if (P.msk[e]) {
        ++present;
        only = P.cls[e];
        if (P.msk[e] & 1) k0 = P.cls[e];
      }
    if (present == 1) {
      P.axis = 0;
      P.ucls = only;
      return P;
    }
    const double e0 = __ldg(s.pal + k0), r0 = __ldg(s.rpal + k0);
    bool raw = true, rounded = true;
#pragma unroll
    for (int e = 0; e < kProfCls; ++e)
      if (P.msk[e]) {
        raw &= P.cls[e] == k0 || eps_equal(__ldg(s.pal + P.cls[e]), e0);
        rounded &= __ldg(s.rpal + P.cls[e]) == r0;
      }
    P.axis = raw || rounded ? 0 : ax;
    return P;
  }
  // slice by slice (rare): the classes of the slice centres (one call site
  // of the classification: code size)
  int k0 = -1;
  bool one = true, raw = true, rounded = true;
#pragma unroll 1
  for (int t = 0; t < n; ++t) {
    const int k = prof_class(s, P, c, h, n, t);
    if (k < 0) {
      P.axis = -2;
      return P;
    }
    if (scls) scls[t] = static_cast<uint16_t>(k);
    if (t == 0) {
      k0 = k;
      continue;
    }
    one &= k == k0;
    raw &= k == k0 || eps_equal(__ldg(s.pal + k), __ldg(s.pal + k0));
    rounded &= __ldg(s.rpal + k) == __ldg(s.rpal + k0);
  }
  if (one) P.ucls = k0;
  P.axis = raw || rounded ? 0 : ax;
  return P;
}

// multiply-xorshift over the layer bit patterns, one full mix at the end
__host__ __device__ __forceinline__ uint64_t key_step(uint64_t h, uint64_t w) {
  h = (h ^ w) * 0x9E3779B97F4A7C15ull;
  return h ^ (h >> 29);
}
// table lookup of key (n, axis, layer(t)); entry index or -1
template <class L>
__device__ int sgf_find(const DSgf& T, int n, int axis, L layer) {
  if (T.cap == 0) return -1;
  uint64_t h = (static_cast<uint64_t>(n) << 8) ^ static_cast<uint64_t>(axis);  // key_hash
#pragma unroll 1
  for (int t = 0; t < n; ++t) h = key_step(h, static_cast<uint64_t>(__double_as_longlong(layer(t))));
  h = sm64_mix(h);
  for (int i = static_cast<int>(h & (T.cap - 1));; i = (i + 1) & (T.cap - 1)) {
    const int e = __ldg(T.entry + i);
    if (e < 0) return -1;
    if (__ldg(T.hash + i) != h || __ldg(T.axis + e) != axis) continue;
    const double* k = T.keys + static_cast<size_t>(e) * NMAX;
    bool eq = true;
#pragma unroll 1
    for (int t = 0; t < n && eq; ++t) eq = __ldg(k + t) == layer(t);
    if (eq) return e;
  }
}

// sample_panel (sgf.cpp:301-308): upper_bound on the inclusive cdf, entered
// through a guide table (Chen & Asau).  guide[b] is the first index whose
// cdf exceeds fl((b/G)*total); since b = floor(u*G) gives b/G <= u exactly
// and rounding is monotone, every earlier index has cdf <= target, so the
// forward scan returns exactly the upper_bound answer.
constexpr int kGuide = 2048;
__device__ int sample_panel(const double* cdf, const int* guide, int count, double u) {
  const double target = u * __ldg(cdf + count - 1);
  int i = __ldg(guide + static_cast<int>(u * kGuide));
  while (i < count && __ldg(cdf + i) <= target) ++i;
  return i == count ? count - 1 : i;
}

template <class L>
__device__ void record_key(DCounters* C, const DMiss& M, int n, int axis, L layer) {
  const unsigned long long m = atomicAdd(&C->nmiss, 1ull);
  if (m < kMissMax) {
    M.axis[m] = axis;
#pragma unroll 1
    for (int t = 0; t < n; ++t) M.layers[m * NMAX + t] = layer(t);
  }
}

// a first transition missed: the walk restarts from scratch once the key is
// in the table (nothing of it was committed)
template <class L>
__device__ void record_miss(DCounters* C, const DMiss& M, int n, int axis, L layer,
                            long long wid) {
  record_key(C, M, n, axis, layer);
  const unsigned long long r = atomicAdd(&C->nretry, 1ull);
  FRW_DCHECK(C, r < 2ull * M.cap);
  M.retry[r] = wid;
}

__device__ __forceinline__ void set_err(DCounters* C, int code) {
  atomicCAS(&C->err, 0ull, static_cast<unsigned long long>(static_cast<unsigned>(-code)));
}



// ---------------------------------------------------------------------------
// voxel-index clipping of the dielectric boxes for a lazy MicroWalk cube
// (microwalk.cpp:25-30 voxel centres; inclusion is closed per axis, so the
// voxels of a box form an index interval on every axis)

__device__ __forceinline__ double vcenter(double c, double h, double p, int i) {
  return c - h + (i + 0.5) * p;  // (c - h) + ((i + 0.5) * p), no contraction
}

// first i in [0, n] with centre(i) >= lo; last i in [-1, n-1] with centre(i) <= hi
// p = 2h/n (the reference's pitch), ip ~ 1/p: the reciprocal only seeds the
// index guesses, which the exact voxel-centre comparisons then correct
__device__ void clip_axis(double c, double h, double p, double ip, int n, double lo, double hi,
                          int* il, int* ih) {
  const double base = c - h;
  int a = static_cast<int>(floor((lo - base) * ip - 0.5));
  a = max(0, min(n, a));
  while (a > 0 && vcenter(c, h, p, a - 1) >= lo) --a;
  while (a < n && vcenter(c, h, p, a) < lo) ++a;
  int b = static_cast<int>(floor((hi - base) * ip - 0.5));
  b = max(-1, min(n - 1, b));
  while (b < n - 1 && vcenter(c, h, p, b + 1) <= hi) ++b;
  while (b >= 0 && vcenter(c, h, p, b) > hi) --b;
  *il = a;
  *ih = b;
}
__device__ void clip_axis(double c, double h, int n, double lo, double hi, int* il, int* ih) {
  const double p = 2.0 * h / n;
  clip_axis(c, h, p, 1.0 / p, n, lo, hi, il, ih);
}

__device__ __forceinline__ int box_lo(uint64_t b, int a) { return static_cast<int>((b >> (8 * a)) & 0xFF); }
__device__ __forceinline__ int box_hi(uint64_t b, int a) { return static_cast<int>((b >> (24 + 8 * a)) & 0xFF); }
__device__ __forceinline__ int box_cls(uint64_t b) { return static_cast<int>((b >> 48) & 0x7FFF); }
// conductor boxes (MicroWalk-E cubes) carry bit 63 and their declaration
// index in bits 48..62; a voxel inside any conductor box is conductor
// (first declared wins, geometry.cpp:57-62 with tol 0), class code kCond
constexpr int kCond = 0xFE;
constexpr int kFace = 0xFF;
__device__ __forceinline__ bool box_is_cond(uint64_t b) { return (b >> 63) != 0; }
__device__ __forceinline__ int box_cond(uint64_t b) { return static_cast<int>((b >> 48) & 0x7FFF); }
__device__ __forceinline__ uint64_t pack_box(const int lo[3], const int hi[3], uint64_t tag) {
  return static_cast<uint64_t>(lo[0]) | static_cast<uint64_t>(lo[1]) << 8 |
         static_cast<uint64_t>(lo[2]) << 16 | static_cast<uint64_t>(hi[0]) << 24 |
         static_cast<uint64_t>(hi[1]) << 32 | static_cast<uint64_t>(hi[2]) << 40 | tag << 48;
}
__device__ __forceinline__ bool box_has(uint64_t b, int i, int j, int k) {
  return i >= box_lo(b, 0) && i <= box_hi(b, 0) && j >= box_lo(b, 1) && j <= box_hi(b, 1) &&
         k >= box_lo(b, 2) && k <= box_hi(b, 2);
}
// class of voxel (i,j,k): the last clipped box containing it, else background
__device__ int cell_class(const uint64_t* boxes, int K, int bg, int i, int j, int k) {
  int cls = bg;
  bool cond = false;
  for (int q = 0; q < K; ++q) {
    const uint64_t b = boxes[q];
    if (box_has(b, i, j, k)) {
      if (box_is_cond(b))
        cond = true;
      else
        cls = box_cls(b);
    }
  }
  return cond ? kCond : cls;
}

// extent [lo, hi] of the cell segment containing v along axis a
__device__ void cell_extent(const uint64_t* boxes, int K, int n, int a, int v, int* lo, int* hi) {
  int l = 0, r = n - 1;
  for (int q = 0; q < K; ++q) {
    const uint64_t b = boxes[q];
    const int bl = box_lo(b, a), bh = box_hi(b, a);
    if (bl <= v) l = max(l, bl); else r = min(r, bl - 1);
    if (bh < v) l = max(l, bh + 1); else r = min(r, bh);
  }
  *lo = l;
  *hi = r;
}

// node packing: i | j<<8 | k<<16
__device__ __forceinline__ int coord(uint32_t node, int a) { return (node >> (8 * a)) & 0xFF; }

// ---- cell atlas lookups ---------------------------------------------------
__device__ __forceinline__ uint64_t upto(int v) { return (2ull << v) - 1; }  // bits 0..v

// Job-local class of the voxels contained in exactly the clipped boxes of M:
// any conductor box (bits [0, ncond)) makes it conductor, else the last
// declared dielectric box wins (geometry.cpp:42-55) -- local class b + 1 for
// mask bit b, its palette class in the atlas (kAtCls) -- else background,
// local class 0.  Local classes (<= KMAX) keep a cell's seven classes in one
// word whatever the structure's palette size.
__device__ __forceinline__ int class_of(uint64_t M, uint64_t cmask) {
  if (M & cmask) return kCond;
  const uint64_t d = M & ~cmask;
  return d ? 64 - __clzll(d) : 0;
}
// palette class of a job-local class
__device__ __forceinline__ int global_class(const uint64_t* A, int lc, int bg) {
  return lc ? reinterpret_cast<const uint16_t*>(A + kAtCls)[lc - 1] : bg;
}

__device__ __forceinline__ uint64_t cond_mask(int ncond) {
  return ncond >= 64 ? ~0ull : (1ull << ncond) - 1;
}

// box set of the voxel at integer coordinates v
__device__ __forceinline__ uint64_t voxel_mask(const uint64_t* A, const uint64_t bm[3],
                                               const int v[3]) {
  uint64_t M = ~0ull;
#pragma unroll
  for (int a = 0; a < 3; ++a) M &= A[kAtMask + 64 * a + __popcll(bm[a] & upto(v[a])) - 1];
  return M;
}

// ---- cell lookup by a scan of the job's clipped boxes ----------------------
// A lane's clipped boxes are read through a strided view: a shared-memory
// slice (box q of lane t at [q * blockDim + t], conflict-free) when the job
// has at most kBoxSm boxes, else the job entry in global memory.
constexpr int kBoxSm = 16;
constexpr int kBoxSmem512 = 512 * kBoxSm * 8;  // dynamic shared memory of 512- / 256-thread CTAs
constexpr int kBoxSmem256 = 256 * kBoxSm * 8;
struct BoxView {
  const uint64_t* p;
  int stride;
  __device__ __forceinline__ uint64_t operator[](int q) const { return p[q * stride]; }
};

// The cell (maximal box of voxels with one box set) holding `node`, its face
// distances (room, one byte per direction 2a+side) and the classes of the six
// face-neighbour cells (kFace on a lattice face) with its own in byte 6, from
// the boxes themselves (no atlas): along each axis the
// cell is cut by every box face (lo and hi + 1), so its extent is bounded by
// the nearest cut at or below the node and the nearest above; the classes of
// the cell and of the six face-neighbour cells are those of one voxel each
// (the node, and the voxel just across each face), i.e. of the boxes holding
// it: any conductor box -> conductor, else the last declared dielectric box
// (local class q + 1), else background (geometry.cpp:42-62).  Two passes of
// O(K) register work; no atlas, no global memory when the boxes are staged.
__device__ uint64_t cell_scan(const BoxView B, int K, int ncond, int n, uint32_t node,
                              uint64_t* room_out) {
  const int v0 = coord(node, 0), v1 = coord(node, 1), v2 = coord(node, 2);
  int lo0 = 0, lo1 = 0, lo2 = 0, hi0 = n - 1, hi1 = n - 1, hi2 = n - 1;
#pragma unroll 1
  for (int q = 0; q < K; ++q) {
    const uint64_t b = B[q];
#define FRW_CUT(a, v, lo, hi)                              \
  {                                                        \
    const int bl = box_lo(b, a), bh = box_hi(b, a) + 1;    \
    if (bl <= v) lo = max(lo, bl); else hi = min(hi, bl - 1); \
    if (bh <= v) lo = max(lo, bh); else hi = min(hi, bh - 1); \
  }
    FRW_CUT(0, v0, lo0, hi0)
    FRW_CUT(1, v1, lo1, hi1)
    FRW_CUT(2, v2, lo2, hi2)
#undef FRW_CUT
  }
  // box sets of the node and of the voxels across the six faces
  uint64_t M = 0, Ml0 = 0, Mh0 = 0, Ml1 = 0, Mh1 = 0, Ml2 = 0, Mh2 = 0;
#pragma unroll 1
  for (int q = 0; q < K; ++q) {
    const uint64_t b = B[q], bit = 1ull << q;
    const int bl0 = box_lo(b, 0), bh0 = box_hi(b, 0), bl1 = box_lo(b, 1), bh1 = box_hi(b, 1),
              bl2 = box_lo(b, 2), bh2 = box_hi(b, 2);
    const bool i0 = bl0 <= v0 && v0 <= bh0, i1 = bl1 <= v1 && v1 <= bh1,
               i2 = bl2 <= v2 && v2 <= bh2;
    if (i0 && i1 && i2) M |= bit;
    if (i1 && i2) {
      if (bl0 <= lo0 - 1 && lo0 - 1 <= bh0) Ml0 |= bit;
      if (bl0 <= hi0 + 1 && hi0 + 1 <= bh0) Mh0 |= bit;
    }
    if (i0 && i2) {
      if (bl1 <= lo1 - 1 && lo1 - 1 <= bh1) Ml1 |= bit;
      if (bl1 <= hi1 + 1 && hi1 + 1 <= bh1) Mh1 |= bit;
    }
    if (i0 && i1) {
      if (bl2 <= lo2 - 1 && lo2 - 1 <= bh2) Ml2 |= bit;
      if (bl2 <= hi2 + 1 && hi2 + 1 <= bh2) Mh2 |= bit;
    }
  }
  const uint64_t cmask = cond_mask(ncond);
  uint64_t room = 0x0101ull << 48;  // two unused bytes kept non-zero
  room |= static_cast<uint64_t>(v0 - lo0) | static_cast<uint64_t>(hi0 - v0) << 8 |
          static_cast<uint64_t>(v1 - lo1) << 16 | static_cast<uint64_t>(hi1 - v1) << 24 |
          static_cast<uint64_t>(v2 - lo2) << 32 | static_cast<uint64_t>(hi2 - v2) << 40;
  *room_out = room;
  uint64_t fc = static_cast<uint64_t>(class_of(M, cmask)) << 48;
  fc |= static_cast<uint64_t>(lo0 > 0 ? class_of(Ml0, cmask) : kFace);
  fc |= static_cast<uint64_t>(hi0 < n - 1 ? class_of(Mh0, cmask) : kFace) << 8;
  fc |= static_cast<uint64_t>(lo1 > 0 ? class_of(Ml1, cmask) : kFace) << 16;
  fc |= static_cast<uint64_t>(hi1 < n - 1 ? class_of(Mh1, cmask) : kFace) << 24;
  fc |= static_cast<uint64_t>(lo2 > 0 ? class_of(Ml2, cmask) : kFace) << 32;
  fc |= static_cast<uint64_t>(hi2 < n - 1 ? class_of(Mh2, cmask) : kFace) << 40;
  return fc;
}

// the first declared conductor box holding voxel v (-1: none)
__device__ __forceinline__ int cond_box_at(const BoxView B, int ncond, const int v[3]) {
#pragma unroll 1
  for (int q = 0; q < ncond; ++q)
    if (box_has(B[q], v[0], v[1], v[2])) return q;
  return -1;
}

// builds the atlas of the K clipped boxes of a job (compile_mw_job)
__device__ void build_atlas(const uint64_t* boxes, int K, int n, uint64_t* A, uint64_t bm[3]) {
  // register-only scan (an O(K + segments) sweep needs per-segment event
  // arrays in local memory, which cost the walk kernels more than it saved)
#pragma unroll 1
  for (int a = 0; a < 3; ++a) {
    uint64_t b = 1;  // segment starting at 0
#pragma unroll 1
    for (int q = 0; q < K; ++q) {
      const uint64_t x = boxes[q];
      const int h = box_hi(x, a) + 1;
      b |= 1ull << box_lo(x, a);
      if (h < n) b |= 1ull << h;
    }
    bm[a] = b;
    A[kAtBm + a] = b;
    int sg = 0;
    for (uint64_t y = b; y; y &= y - 1, ++sg) {
      const int st = __ffsll(y) - 1;
      uint64_t m = 0;
#pragma unroll 1
      for (int q = 0; q < K; ++q) {
        const uint64_t x = boxes[q];
        if (box_lo(x, a) <= st && st <= box_hi(x, a)) m |= 1ull << q;
      }
      A[kAtMask + 64 * a + sg] = m;
    }
  }
}

// Compiles the MicroWalk job of a cube into job entry `slot`: the boxes that
// reach into the cube clipped to voxel-index ranges (with the reference's
// voxel-centre arithmetic, microwalk.cpp:25-30) and their cell atlas.  With
// `conductors` (MicroWalk-E, microwalk.cpp:206-228) conductor boxes are
// clipped too.  Returns 1 ok, 0 when the start voxel is conductor
// (EngulfedStart), 3 when more than KMAX boxes reach into the cube (only
// the cube is stored: the hop runs on a dense grid, k_mw_dense).
template <bool ATLAS_OK = true>
__device__ int compile_mw_job(const DStruct& s, const DSlots& W, int slot, const double c[3],
                              double h, int n, bool conductors, bool atlas_arg, DCounters* C) {
  const bool atlas = ATLAS_OK && atlas_arg;  // (instantiated without the atlas in k_tail)
  FRW_DCHECK(C, slot >= 0 && slot < W.J);
  uint64_t* boxes = W.boxes + static_cast<size_t>(slot) * KMAX;
  uint64_t* A = W.atlas + static_cast<size_t>(slot) * kAtlasWords;
  int K = 0, ncond = 0;
  const double cb[6] = {c[0] - h, c[1] - h, c[2] - h, c[0] + h, c[1] + h, c[2] + h};
  const double pitch = 2.0 * h / n, ipitch = 1.0 / pitch;
  int cand[kCandMax];
  uint16_t* cls = reinterpret_cast<uint16_t*>(A + kAtCls);
  // phase 0: conductor boxes (MicroWalk-E only), phase 1: dielectric boxes,
  // each in declaration order.  One rolled loop (one inlined copy of the
  // candidate query and the clip): the walk kernels are instruction-fetch
  // bound, and the box-axis work is not on a hot path
#pragma unroll 1
  for (int ph = conductors ? 0 : 1; ph < 2; ++ph) {
    const bool cph = ph == 0;
    if (!cph) ncond = K;
    const int nca = grid_candidates(s, !cph, cb, cand);
    const int ni = nca < 0 ? (cph ? s.nc : s.nd) : nca;
    const double* base = cph ? s.cbox : s.dbox;
#pragma unroll 1
    for (int i = 0; i < ni; ++i) {
      const int q = nca < 0 ? i : cand[i];
      const double* bx = base + 6 * q;
      // voxel centres lie inside the closed cube: a box that misses the
      // cube cannot contain one (cheap reject before the exact clip).  All
      // six compares, no short-circuit: lanes scanning different boxes stay
      // on one path (the || chain split warps six ways, 2.5 active lanes on C4)
      double b6[6];
#pragma unroll
      for (int e = 0; e < 6; ++e) b6[e] = __ldg(bx + e);
      if ((b6[0] > cb[3]) | (b6[3] < cb[0]) | (b6[1] > cb[4]) | (b6[4] < cb[1]) |
          (b6[2] > cb[5]) | (b6[5] < cb[2]))
        continue;
      uint64_t pk = 0;  // pack_box layout: lo bytes 0-2, hi bytes 3-5
      bool empty = false;
#pragma unroll 1
      for (int ax = 0; ax < 3; ++ax) {
        const double ca = ax == 0 ? c[0] : (ax == 1 ? c[1] : c[2]);
        int l, hh;
        clip_axis(ca, h, pitch, ipitch, n, __ldg(bx + ax), __ldg(bx + 3 + ax), &l, &hh);
        empty |= l > hh;
        pk |= static_cast<uint64_t>(l & 0xFF) << (8 * ax) |
              static_cast<uint64_t>(hh & 0xFF) << (24 + 8 * ax);
      }
      if (empty) continue;
      if (K == KMAX) {
        // more than KMAX boxes reach into the cube: the hop runs on a dense
        // voxel-class grid (k_mw_dense); EngulfedStart from the start
        // voxel's centre (microwalk.cpp:83-86: a conductor holds it)
        if (conductors) {
          const int m = (n - 1) / 2;
          const double pitch = 2.0 * h / n;
          const double p0[3] = {vcenter(c[0], h, pitch, m), vcenter(c[1], h, pitch, m),
                                vcenter(c[2], h, pitch, m)};
          if (conductor_at(s, p0, 0.0) >= 0) return 0;
        }
        W.cube[4 * slot + 0] = c[0];
        W.cube[4 * slot + 1] = c[1];
        W.cube[4 * slot + 2] = c[2];
        W.cube[4 * slot + 3] = h;
        return 3;
      }
      if (cph) {
        boxes[K++] = pk | (0x8000ull | static_cast<uint64_t>(q)) << 48;
      } else {
        const int dc = __ldg(s.dcls + q);
        if (atlas) cls[K] = static_cast<uint16_t>(dc);
        boxes[K++] = pk | static_cast<uint64_t>(dc) << 48;
      }
    }
  }
  // the cell atlas only for FDM jobs (k_fdm classifies voxels from it); the
  // MicroWalk kernels look cells up by scanning the boxes (cell_scan)
  if (atlas) {
    uint64_t bm[3];
    build_atlas(boxes, K, n, A, bm);
  }
  const int m = (n - 1) / 2;  // start_node (sgf.hpp:58-61)
  const int v0[3] = {m, m, m};
  // EngulfedStart (microwalk.cpp:83-86): a conductor box holds the start
  // voxel.  The start cell itself is looked up by the first super-step.
  if (ncond && cond_box_at(BoxView{boxes, 1}, ncond, v0) >= 0) return 0;
  W.nbox[slot] = static_cast<uint16_t>(ncond | K << 8);
  W.cube[4 * slot + 0] = c[0];
  W.cube[4 * slot + 1] = c[1];
  W.cube[4 * slot + 2] = c[2];
  W.cube[4 * slot + 3] = h;
  return 1;
}

// ---------------------------------------------------------------------------
// first transition (engine.cpp:201-288); returns 1 ok, 0 degenerate point,
// 2 table miss (key recorded), <0 error

struct FirstOut {
  double p[3];
  double weight;
  int branch;
};

__device__ int first_transition(const DStruct& s, const DSgf& T, const DParams& P, long long wid,
                                Rng& rng, const double g[3], int gaxis, int gsign,
                                uint64_t* boxes, DCounters* C, const DMiss& M, FirstOut* out) {
  if (conductor_at(s, g, P.snap) >= 0) return 0;
  double fh;
  if (!max_free_cube(s, g, &fh)) return -1;
  if (!(fh > P.snap)) return 0;
  const int n = P.n;
  double c[3], h;
  transit_cube(g, fh, n, c, &h);
  double layers[NMAX];
  bool own_layers = false;  // ladder branches 2-3 build the layers themselves
  int branch = 0;
  Prof pr = strat_probe(s, c, h, n);
  int axis = pr.axis;
  if (axis == -2) return -1;
  if (axis < 0) {
    for (int i = 19; i >= 6; --i) {  // concentric shrink, engine.cpp:218-226
      double c2[3], h2;
      transit_cube(g, 0.05 * i * fh, n, c2, &h2);
      pr = strat_probe(s, c2, h2, n);
      axis = pr.axis;
      if (axis == -2) return -1;
      if (axis >= 0) {
        c[0] = c2[0];
        c[1] = c2[1];
        c[2] = c2[2];
        h = h2;
        branch = 1;
        break;
      }
    }
  }
  if (axis < 0) {
    // build_grid + slice means (engine.cpp:228-265), summed in the
    // reference's loop order so the means are bit-identical
    int K = 0;
    int cand[kCandMax];
    const double cb[6] = {c[0] - h, c[1] - h, c[2] - h, c[0] + h, c[1] + h, c[2] + h};
    const int dcand = grid_candidates(s, true, cb, cand);
    for (int i = 0, ni = dcand < 0 ? s.nd : dcand; i < ni; ++i) {
      const int d = dcand < 0 ? i : cand[i];
      const double* b = s.dbox + 6 * d;
      if ((__ldg(b) > c[0] + h) | (__ldg(b + 3) < c[0] - h) | (__ldg(b + 1) > c[1] + h) |
          (__ldg(b + 4) < c[1] - h) | (__ldg(b + 2) > c[2] + h) | (__ldg(b + 5) < c[2] - h))
        continue;
      int lo[3], hi[3];
      bool empty = false;
      for (int a = 0; a < 3; ++a) {
        clip_axis(c[a], h, n, __ldg(b + a), __ldg(b + 3 + a), &lo[a], &hi[a]);
        empty |= lo[a] > hi[a];
      }
      if (empty) continue;
      if (K == KMAX) {  // more boxes than the list holds: classify voxel centres
        K = -1;
        break;
      }
      boxes[K++] = pack_box(lo, hi, static_cast<uint64_t>(__ldg(s.dcls + d)));
    }
    double sl[3][NMAX];
    for (int a = 0; a < 3; ++a)
      for (int t = 0; t < n; ++t) sl[a][t] = 0.0;
    const double pitch = 2.0 * h / n;
    for (int k = 0; k < n; ++k)
      for (int j = 0; j < n; ++j) {
        // the class is constant between x-breakpoints: walk the row by cells
        int i = 0;
        while (i < n) {
          int lo, hi;
          double e;
          if (K >= 0) {
            cell_extent(boxes, K, n, 0, i, &lo, &hi);
            e = __ldg(s.pal + cell_class(boxes, K, s.bg, i, j, k));
          } else {  // permittivity_at(voxel_center) (geometry.cpp:320-349)
            const double pv[3] = {vcenter(c[0], h, pitch, i), vcenter(c[1], h, pitch, j),
                                  vcenter(c[2], h, pitch, k)};
            lo = hi = i;
            e = __ldg(s.pal + eps_class_at(s, pv));
          }
          for (; i <= hi; ++i) {
            sl[0][i] += e;
            sl[1][j] += e;
            sl[2][k] += e;
          }
        }
      }
    int best = 0;
    double bvar = -1.0;
    for (int a = 0; a < 3; ++a) {
      double mean = 0;
      for (int t = 0; t < n; ++t) {
        sl[a][t] /= static_cast<double>(n) * n;
        mean += sl[a][t];
      }
      mean /= n;
      double var = 0;
      for (int t = 0; t < n; ++t) var += (sl[a][t] - mean) * (sl[a][t] - mean);
      if (var > bvar) {
        bvar = var;
        best = a;
      }
    }
    axis = best;
    bool same = true;
    for (int t = 0; t < n; ++t) {
      layers[t] = round_sig6(sl[best][t]);
      same &= layers[t] == layers[0];
    }
    branch = 2;
    if (same) {
      branch = 3;
      axis = 0;
    }
    own_layers = true;
  }
  auto layer = [&](int t) { return own_layers ? layers[t] : prof_layer(s, pr, c, h, n, t); };
  int e = !own_layers && pr.ucls >= 0 ? __ldg(T.uentry + pr.ucls) : -1;
  if (e < 0) e = sgf_find(T, n, axis, layer);
  if (e < 0) {
    record_miss(C, M, n, axis, layer, wid);
    return 2;
  }
  const double* data = T.data[e];
  const int panels = P.panels;
  const int panel = sample_panel(data, reinterpret_cast<const int*>(data + 5 * panels), panels,
                                 uniform(P, wid, rng));
  const double pitch_nm = 2.0 * h / n;
  const double kern_per_m =
      __ldg(data + 2 * panels + gaxis * panels + panel) * (__ldg(T.pitch + e) / pitch_nm) /
      kMPerNm;
  const int ecls = eps_class_at(s, g);
  if (ecls < 0) return -1;
  const double eps_r = __ldg(s.pal + ecls);
  panel_center(c, h, n, panel, out->p);
  out->weight = -P.area * kEps0 * eps_r * gsign * kern_per_m / __ldg(data + panels + panel);
  out->branch = branch;
  return 1;
}

// ---------------------------------------------------------------------------
// kernels

__device__ void finish_walk(const DSlots& W, WalkRec* recs, DCounters* C, int slot, int term,
                            bool aborted) {
  const long long wid = W.wid[slot];
  WalkRec r;
  r.weight = W.weight[slot];
  r.mw_steps = W.mwsteps[slot];
  r.slot = term;
  r.cached = W.cached[slot];
  r.mw = W.mw[slot];
  r.aborted = aborted;
  r.branch = W.branch[slot];
  r.resampled = W.resampled[slot];
  r.done = 1;
  FRW_DCHECK(C, wid >= 0 && wid < W.count);
  recs[wid] = r;
  W.state[slot] = S_FREE;
  atomicAdd(&C->done, 1ull);
#ifdef FRW_PHASE_CLOCKS
  if (g_in_tail) {
    const unsigned long long dt = (gtimer() - g_tail_t0) / 250000ull;
    atomicAdd(&g_tail_hist[dt < 255 ? dt : 255], 1ull);
  }
#endif
}

// Gaussian sample + first transition for every free slot
__global__ void k_spawn(DStruct s, DSgf T, DParams P, DSlots W, WalkRec* recs, DCounters* C,
                        DMiss M, int* aq) {
  for (int slot = blockIdx.x * blockDim.x + threadIdx.x; slot < W.S;
       slot += gridDim.x * blockDim.x) {
    if (W.state[slot] != S_FREE) continue;
    long long wid = -1;
    if (C->pend_head < C->npend) {
      const unsigned long long q = atomicAdd(&C->pend_head, 1ull);
      if (q < C->npend) wid = M.pend[q];
    }
    if (wid < 0) {
      if (C->next >= static_cast<unsigned long long>(P.count)) continue;
      const unsigned long long q = atomicAdd(&C->next, 1ull);
      if (q >= static_cast<unsigned long long>(P.count)) continue;
      wid = static_cast<long long>(q);
    }
    Rng rng;
    rng.s = P.rng == FRW_RNG_SPLITMIX_PARITY
                ? sm64_stream_from_mixed(P.mixed_seed, P.walk_begin + wid)
                : 0;
    W.wid[slot] = wid;
    W.cached[slot] = 0;
    W.mw[slot] = 0;
    W.mwsteps[slot] = 0;
    W.hops[slot] = 0;
    FirstOut fo;
    int rc = 0, resampled = 0;
    for (int attempt = 0; attempt < 100 && rc == 0; ++attempt) {  // engine.cpp:359-363
      // sample_gaussian (engine.cpp:126-148)
      const double u = uniform(P, wid, rng);
      int face = 5;
      for (int f = 0; f < 5; ++f)
        if (u < P.fcdf[f]) {
          face = f;
          break;
        }
      const int a = face >> 1;
      const int b1 = a == 0 ? 1 : 0;
      const int b2 = a == 2 ? 1 : 2;
      const int sign = ((face & 1) ? 1 : -1);
      double g[3];
      g[a] = sign < 0 ? P.gbox[a] : P.gbox[3 + a];
      g[b1] = P.gbox[b1] + uniform(P, wid, rng) * (P.gbox[3 + b1] - P.gbox[b1]);
      g[b2] = P.gbox[b2] + uniform(P, wid, rng) * (P.gbox[3 + b2] - P.gbox[b2]);
      PH_T0(ph8);
      rc = first_transition(s, T, P, wid, rng, g, a, sign,
                            W.boxes + static_cast<size_t>(slot) * KMAX, C, M, &fo);
      PH_ADD(8, ph8);
      if (rc == 0) ++resampled;
    }
    W.resampled[slot] = static_cast<uint8_t>(resampled);
    if (rc < 0) {
      set_err(C, FRW_EINVAL);
      continue;
    }
    if (rc == 2) continue;  // miss: parked for a restart, slot stays free
    if (rc == 0) {          // resample cap: folded into ground as aborted
      W.weight[slot] = 0.0;
      W.branch[slot] = 0xFF;
      finish_walk(W, recs, C, slot, s.nc, true);
      continue;
    }
    W.p[3 * slot + 0] = fo.p[0];
    W.p[3 * slot + 1] = fo.p[1];
    W.p[3 * slot + 2] = fo.p[2];
    W.weight[slot] = fo.weight;
    W.branch[slot] = static_cast<uint8_t>(fo.branch);
    W.rng[slot] = rng.s;
    W.state[slot] = S_ACTIVE;
    const unsigned long long qa = atomicAdd(&C->alen, 1ull);
    FRW_DCHECK(C, qa < static_cast<unsigned long long>(W.S));
    aq[qa] = slot;
  }
}

// Lane-held state of a walk in the advance stage.
struct AdvLane {
  int slot;
  int jslot;     // job entry a compiled MicroWalk hop goes to (the slot, or
                 // in k_tail the lane's own L2-resident entry)
  long long wid;
  double p[3];
  Rng rng;
  int hops;
  uint32_t cached;
};

__device__ __forceinline__ void adv_load(const DSlots& W, int slot, AdvLane& L) {
  L.slot = slot;
  L.jslot = slot;
  L.wid = W.wid[slot];
  L.p[0] = W.p[3 * slot];
  L.p[1] = W.p[3 * slot + 1];
  L.p[2] = W.p[3 * slot + 2];
  L.rng.s = W.rng[slot];
  L.hops = W.hops[slot];
  L.cached = W.cached[slot];
}

// The MicroWalk job of a general cube (engine.cpp:311-347) at point p with
// free-cube half width fh: MicroWalk on the transit cube, or MicroWalk-E on
// the expanded cube, falling back to the transit cube when the expanded
// lattice swallows the start voxel (EngulfedStart).  Compiled into job entry
// jslot.  Returns 2 (job ready, its kind in W.mwkind[jslot]) or 1 (the walk
// left the stage: queued for a dense hop, or dropped on an error).
template <bool ATLAS = true>  // false: never an FDM job (the atlas code is not instantiated)
__device__ __forceinline__ int hop_compile(const DStruct& s, const DParams& P, const DSlots& W,
                                           DCounters* C, const DMiss& M, int slot, int jslot,
                                           const double p[3], double fh) {
  const int n = P.n;
  double c[3], h;
  transit_cube(p, fh, n, c, &h);
  uint8_t kind = P.mode == FRW_MODE_FDM ? 2 : 0;  // 2: FDM solve (engine.cpp:311-318)
  double jc[3] = {c[0], c[1], c[2]}, jh = h;
  bool expanded = false;
  if (P.mode == FRW_MODE_MWE || P.mode == FRW_MODE_HYBRID_MWE) {
    kind = 1;
    expanded = true;
    const double wall = cheb_wall(s.world, p);
    const double half = mn(P.expansion * fh, wall);  // microwalk.cpp:213-214
    if (!(half > 0)) {
      set_err(C, FRW_EINVAL);
      W.state[slot] = S_FREE;
      return 1;
    }
    transit_cube(p, half, n, jc, &jh);
  }
  // one inlined copy of the job compiler (the kernels are instruction-fetch
  // bound): the expanded cube first, the transit cube on EngulfedStart
  int rc = -1;
#pragma unroll 1
  for (;;) {
    rc = compile_mw_job<ATLAS>(s, W, jslot, jc, jh, n, expanded, kind == 2, C);
    if (rc != 0 || !expanded) break;
    expanded = false;
    jc[0] = c[0];
    jc[1] = c[1];
    jc[2] = c[2];
    jh = h;
  }
  if (rc < 0) {
    W.state[slot] = S_FREE;
    return 1;
  }
  if (rc == 3) {
    // more than KMAX boxes reach into the cube: the hop goes to k_mw_dense
    // (its job in the walk's own entry: the dense kernel runs after this one)
    if (kind == 2) {  // FDM builds its system from the atlas
      set_err(C, FRW_EINVAL);
      W.state[slot] = S_FREE;
      return 1;
    }
    if (jslot != slot) {
#pragma unroll
      for (int q = 0; q < 4; ++q) W.cube[4 * slot + q] = W.cube[4 * jslot + q];
    }
    W.mwkind[slot] = static_cast<uint8_t>(kind | kDense | (expanded ? kDenseCond : 0));
    const unsigned long long qd = atomicAdd(&C->dqlen, 1ull);
    FRW_DCHECK(C, qd < static_cast<unsigned long long>(W.S));
    M.dense[qd] = slot;
    return 1;
  }
  W.mwkind[jslot] = kind;
  return 2;
}

// One transition (engine.cpp:290-350; hop cap engine.cpp:367-375) of the
// lane's walk.  Returns 0 when a cached hop was taken (the walk stays with
// the lane), 1 when the walk left the stage (terminated or parked by a
// table miss), 2 when its walk needs a MicroWalk hop: with a compile queue
// `cq` (wavefront rounds) the walk is queued for k_compile, else its job is
// compiled here into the lane's job entry.
// QUEUE: the compile queue is always given (k_advance), so the inline job
// compiler is not instantiated there
template <bool QUEUE = false, bool ATLAS = true>
__device__ int advance_once(const DStruct& s, const DSgf& T, const DParams& P, const DSlots& W,
                            WalkRec* recs, DCounters* C, const DMiss& M, int* cq, AdvLane& L) {
  const int slot = L.slot;
  const int n = P.n;
  if (L.hops >= P.hop_cap) {
    W.cached[slot] = L.cached;
    finish_walk(W, recs, C, slot, s.nc, true);
    return 1;
  }
  double fh;
  PH_T0(ph0);
  const int g = hop_scan(s, L.p, P.snap, &fh);
  PH_ADD(0, ph0);
  if (g >= 0 || g == -1) {  // snapped to a conductor / to the grounded wall
    W.cached[slot] = L.cached;
    finish_walk(W, recs, C, slot, g >= 0 ? g : s.nc, false);
    return 1;
  }
  if (g == -2) {
    set_err(C, FRW_EINVAL);
    W.state[slot] = S_FREE;
    return 1;
  }
  double c[3], h;
  transit_cube(L.p, fh, n, c, &h);
  PH_T0(ph1);
  uint16_t scls[NMAX];  // slice classes of an overflowing profile (rare; local memory)
  const Prof pr = strat_probe(s, c, h, n, scls);
  PH_ADD(1, ph1);
  const int axis = pr.axis;
  if (axis == -2) {
    set_err(C, FRW_EINVAL);
    W.state[slot] = S_FREE;
    return 1;
  }
  if (axis >= 0) {
    // a single-class cube (2/3 of the cached hops on C3/C5) finds its entry
    // through the per-class uniform index; otherwise (or when that key is
    // not in the table yet) the full key is hashed and compared
    // the rounded layer values of the profile's (class, slice-mask) pairs
    // in registers: a layer is four mask tests, no palette load per slice
    double lv[kProfCls];
#pragma unroll
    for (int q = 0; q < kProfCls; ++q) lv[q] = pr.msk[q] ? __ldg(s.rpal + pr.cls[q]) : 0.0;
    auto layer = [&](int t) {
      if (pr.ucls >= 0) return __ldg(s.rpal + pr.ucls);
      if (pr.ovf) return __ldg(s.rpal + scls[t]);
      double x = 0.0;
#pragma unroll
      for (int q = 0; q < kProfCls; ++q)
        if ((pr.msk[q] >> t) & 1) x = lv[q];
      return x;
    };
    PH_T0(ph2);
    int e = pr.ucls >= 0 ? __ldg(T.uentry + pr.ucls) : -1;
    if (e < 0) e = sgf_find(T, n, axis, layer);
    if (e < 0) {
      // parked mid-walk: the key is looked up before any draw, so the walk
      // resumes from this state, bit-identical to an uninterrupted run
      record_key(C, M, n, axis, layer);
      W.p[3 * slot] = L.p[0];
      W.p[3 * slot + 1] = L.p[1];
      W.p[3 * slot + 2] = L.p[2];
      W.rng[slot] = L.rng.s;
      W.hops[slot] = L.hops;
      W.cached[slot] = L.cached;
      W.state[slot] = S_PARKED;
      const unsigned long long qp = atomicAdd(&C->npark, 1ull);
      FRW_DCHECK(C, qp < 2ull * M.cap);
      M.park[qp] = slot;
      return 1;
    }
    const double* data = T.data[e];
    const int panel = sample_panel(data, reinterpret_cast<const int*>(data + 5 * P.panels),
                                   P.panels, uniform(P, L.wid, L.rng));
    panel_center(c, h, n, panel, L.p);
    PH_ADD(2, ph2);
    ++L.cached;
    ++L.hops;
    return 0;
  }
  // general cube (engine.cpp:311-347): the walk waits for its MicroWalk hop
  W.p[3 * slot + 0] = L.p[0];
  W.p[3 * slot + 1] = L.p[1];
  W.p[3 * slot + 2] = L.p[2];
  W.rng[slot] = L.rng.s;
  W.hops[slot] = L.hops + 1;
  W.cached[slot] = L.cached;
  W.state[slot] = S_NEED_MW;
  if (QUEUE || cq) {
    // wavefront rounds: k_compile builds the job, every lane of a warp
    // compiling one (in k_advance only a few lanes of a warp would, the rest
    // waiting: the job compiler was over half of k_advance's issue slots at
    // 2.6 active lanes)
    W.cube[4 * slot + 3] = fh;
    const unsigned long long qc = atomicAdd(&C->cqlen, 1ull);
    FRW_DCHECK(C, qc < static_cast<unsigned long long>(W.S));
    cq[qc] = slot;
    return 2;
  }
  PH_T0(ph3);
  const int rc = hop_compile<ATLAS>(s, P, W, C, M, slot, L.jslot, L.p, fh);
  PH_ADD(3, ph3);
  return rc;
}

// (FRW_DEBUG_CHECKS) the lane's node lies in the lattice
__device__ __forceinline__ bool node_ok(uint32_t node, int n) {
  return coord(node, 0) < n && coord(node, 1) < n && coord(node, 2) < n;
}

// the walk goes back to the next round's ACTIVE queue
__device__ __forceinline__ void mw_requeue(DCounters* C, int* aq_out, int slot) {
  aq_out[atomicAdd(&C->a2len, 1ull)] = slot;  // (checked by the host: a2len <= S)
}

// persistent: each thread takes ACTIVE walks from the queue and advances
// them one transition per iteration, re-armed as soon as its walk leaves.
// The grid is 4 x 256 threads per SM, so registers must allow 4 CTAs
#ifndef FRW_ADV_MINB
#define FRW_ADV_MINB 4
#endif
__global__ void __launch_bounds__(256, FRW_ADV_MINB)
    k_advance(DStruct s, DSgf T, DParams P, DSlots W, WalkRec* recs, DCounters* C, DMiss M,
              const int* aq, int* cq, int* aq_out) {
  const unsigned long long alen = C->alen;
  const int slice = P.adv_slice > 0 ? P.adv_slice : 0x7FFFFFFF;
  unsigned long long item = atomicAdd(&C->ahead, 1ull);
  bool live = item < alen;
  AdvLane L;
  if (live) {
    FRW_DCHECK(C, aq[item] >= 0 && aq[item] < W.S);
    adv_load(W, aq[item], L);
  }
  int left = slice;  // transitions left in this visit of the walk
  while (__any_sync(0xFFFFFFFFu, live)) {
    if (!live) continue;
    int r = advance_once<true>(s, T, P, W, recs, C, M, cq, L);
    if (r == 0 && --left == 0) {
      // a long chain of cached hops: the walk continues next round
      W.p[3 * L.slot] = L.p[0];
      W.p[3 * L.slot + 1] = L.p[1];
      W.p[3 * L.slot + 2] = L.p[2];
      W.rng[L.slot] = L.rng.s;
      W.hops[L.slot] = L.hops;
      W.cached[L.slot] = L.cached;
      mw_requeue(C, aq_out, L.slot);
      r = 1;
    }
    if (r != 0) {
      left = slice;
      item = atomicAdd(&C->ahead, 1ull);
      live = item < alen;
      if (live) adv_load(W, aq[item], L);
    }
  }
}

// the MicroWalk jobs of the walks k_advance queued, one per thread (each
// warp compiles 32 jobs side by side), appended to the round's MicroWalk
// queue (or the dense-hop queue)
__global__ void __launch_bounds__(256, 2)
    k_compile(DStruct s, DParams P, DSlots W, DCounters* C, DMiss M, const int* cq, int* mq) {
  const unsigned long long len = C->cqlen;
  for (unsigned long long i = blockIdx.x * blockDim.x + threadIdx.x; i < len;
       i += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
    const int slot = cq[i];
    FRW_DCHECK(C, slot >= 0 && slot < W.S);
    const double p[3] = {W.p[3 * slot], W.p[3 * slot + 1], W.p[3 * slot + 2]};
    const double fh = W.cube[4 * slot + 3];
    if (hop_compile(s, P, W, C, M, slot, slot, p, fh) == 2) {
      const unsigned long long qm = atomicAdd(&C->qlen, 1ull);
      FRW_DCHECK(C, qm < static_cast<unsigned long long>(W.S));
      mq[qm] = slot;
    }
  }
}

// between rounds: the next round's ACTIVE queue becomes current, and the
// MicroWalk hops carried over open the next round's MicroWalk queue
__global__ void k_round(DCounters* C) {
  C->alen = C->a2len;
  C->ahead = 0;
  C->a2len = 0;
  C->qlen = C->q2len;
  C->qhead = 0;
  C->q2len = 0;
  C->dqlen = 0;
  C->dqhead = 0;
  C->cqlen = 0;
}

// ---------------------------------------------------------------------------
// the lazy MicroWalk hop (microwalk.cpp:77-156 with LazyField)

struct MwLane {
  int slot;
  int jslot;      // the hop's job entry (compile_mw_job)
  long long wid;
  uint32_t node;
  uint64_t room;  // distance to the cell faces, one byte per direction
  uint64_t fc;    // face-neighbour classes (byte per dir), current class in byte 6
  uint64_t rng;   // SplitMix64 state or Philox block counter
  int steps;
  int ncond;      // conductor boxes of the job (boxes [0, ncond))
  int nbx;        // clipped boxes of the job
  int hom;        // homogeneous radius known at node hnode (0: none)
  uint32_t hnode;
  int hq;         // the clipped box that limited it (-1: the lattice), see mw_superstep
  BoxView bx;     // the job's clipped boxes (shared-memory slice or job entry)
  double al[6];   // alpha of the neighbour across each face of the cell
  uint32_t gsteps;  // diagnostics, accumulated across the lane's hops
  uint32_t cchg;
  uint32_t jumps;
  uint32_t jsteps;  // steps the lane's jumps stand for
};

// Tables of the MicroWalk kernels: the palette-pair alphas (Pn <= PMAX: in
// shared memory, alpha 1 for absorbing faces at index Pn*Pn) or, for larger
// palettes, the palette itself (alphas divided out, the same IEEE division
// the table holds: e_nb / (e_nb + e_self), microwalk.cpp:97-104).
struct AlphaTab {
  const double* tab;  // smem pair table, or null
  const double* pal;  // palette (global)
  int Pn, bg;
};

// the per-face alphas of the lane's cell: palette pair (face class, own
// class), 1 for lattice and conductor faces (both absorb the step)
// global -> shared 8-byte asynchronous copy (cp.async, sm_80+)
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// palette class of a job-local class (0: background, q + 1: dielectric box q)
__device__ __forceinline__ int lane_class(const MwLane& L, int lc, int bg) {
  return lc ? box_cls(L.bx[lc - 1]) : bg;
}
__device__ __forceinline__ void lane_alphas(const AlphaTab& T, MwLane& L) {
  const int g0 = lane_class(L, static_cast<int>((L.fc >> 48) & 0xFF), T.bg);
  if (T.tab) {
#pragma unroll
    for (int d = 0; d < 6; ++d) {
      const int cn = static_cast<int>((L.fc >> (8 * d)) & 0xFF);
      L.al[d] = T.tab[cn >= kCond ? T.Pn * T.Pn : lane_class(L, cn, T.bg) * T.Pn + g0];
    }
  } else {
    const double e0 = __ldg(T.pal + g0);
#pragma unroll
    for (int d = 0; d < 6; ++d) {
      const int cn = static_cast<int>((L.fc >> (8 * d)) & 0xFF);
      const double en = cn >= kCond ? 0.0 : __ldg(T.pal + lane_class(L, cn, T.bg));
      L.al[d] = cn >= kCond ? 1.0 : en / (en + e0);
    }
  }
}

__device__ __forceinline__ const uint64_t* lane_atlas(const DSlots& W, int slot) {
  return W.atlas + static_cast<size_t>(slot) * kAtlasWords;
}

// bsm: the kernel's shared-memory box slices (kBoxSm per thread, strided by
// blockDim), or null: jobs with at most kBoxSm boxes are staged there
__device__ __forceinline__ void mw_arm(const DSlots& W, int slot, int jslot, int n, MwLane& L,
                                       uint64_t* bsm) {
  const int m = (n - 1) / 2;
  L.slot = slot;
  L.jslot = jslot;
  L.wid = W.wid[slot];
  L.node = m | (m << 8) | (m << 16);
  L.room = 0;  // cell pending: the first super-step looks it up
  L.rng = W.rng[slot];
  {
    const int nb = W.nbox[jslot];
    L.ncond = nb & 0xFF;
    L.nbx = nb >> 8;
  }
  L.hom = 0;
  L.hq = -1;
  {
    const uint64_t* G = W.boxes + static_cast<size_t>(jslot) * KMAX;
    if (bsm && L.nbx <= kBoxSm) {
      uint64_t* d = bsm + threadIdx.x;
      // asynchronous copies (LDGSTS): the loads go out back to back and no
      // register waits on them until the one wait below
#pragma unroll 1
      for (int q = 0; q < L.nbx; ++q) cp_async8(d + q * blockDim.x, G + q);
      // the job's cube (centre, half width) in the slice's top words when it
      // has room: the surface exit then reads no global memory
      if (L.nbx <= kBoxSm - 4) {
        const uint64_t* cube = reinterpret_cast<const uint64_t*>(W.cube) + 4 * static_cast<size_t>(jslot);
#pragma unroll
        for (int q = 0; q < 4; ++q) cp_async8(d + (kBoxSm - 4 + q) * blockDim.x, cube + q);
      }
      cp_async_wait_all();
      L.bx = BoxView{d, static_cast<int>(blockDim.x)};
    } else {
      L.bx = BoxView{G, 1};
    }
  }
  L.steps = 0;
  L.hnode = L.node;
  if (W.state[slot] == S_MW_CARRY) {  // a hop carried over from the last round
    L.node = W.mwnode[slot];
    L.steps = W.mwhsteps[slot];
    const uint64_t hj = W.mwhj[slot];  // the jump decisions continue exactly
    L.hom = static_cast<int>(hj & 0xFF);
    L.hq = static_cast<int>((hj >> 8) & 0xFF) - 1;
    L.hnode = static_cast<uint32_t>(hj >> 32);
  }
}

// the hop's time slice ran out: its state goes to the slot and the job to
// the next round's MicroWalk queue (the stream position is saved, so the
// hop continues bit-identically)
__device__ __forceinline__ void mw_carry(const DSlots& W, DCounters* C, int* mq_next, MwLane& L) {
  W.mwnode[L.slot] = L.node;
  W.mwhsteps[L.slot] = L.steps;
  W.mwhj[L.slot] = static_cast<uint32_t>(L.hom & 0xFF) | static_cast<uint64_t>(L.hq + 1) << 8 |
                   static_cast<uint64_t>(L.hnode) << 32;
  W.rng[L.slot] = L.rng;
  W.state[L.slot] = S_MW_CARRY;
  const unsigned long long qn = atomicAdd(&C->q2len, 1ull);
  FRW_DCHECK(C, qn < static_cast<unsigned long long>(W.S));
  mq_next[qn] = L.slot;
}

// a move left the current cell: look the new cell up from the job's boxes
__device__ __forceinline__ void mw_cell_change(const AlphaTab& T, int n, MwLane& L) {
  L.fc = cell_scan(L.bx, L.nbx, L.ncond, n, L.node, &L.room);
  lane_alphas(T, L);
}

// surface exit: continuation point, counters, slot back to ACTIVE
__device__ void mw_exit(const DSlots& W, int n, MwLane& L, int dir) {
  const int a = dir >> 1;
  const int i = coord(L.node, 0), j = coord(L.node, 1), k = coord(L.node, 2);
  const int u = a == 0 ? j : i;
  const int v = a == 2 ? j : k;
  const int panel = (dir * n + v) * n + u;  // surface_panel_of (sgf.cpp:13-30)
  // the cube from the lane's shared-memory slice when mw_arm staged it there
  const bool staged = L.bx.stride != 1 && L.nbx <= kBoxSm - 4;
  const double* cs = staged ? reinterpret_cast<const double*>(L.bx.p) : W.cube + 4 * L.jslot;
  const int cst = staged ? L.bx.stride : 1, c0 = staged ? kBoxSm - 4 : 0;
  const double c[3] = {cs[c0 * cst], cs[(c0 + 1) * cst], cs[(c0 + 2) * cst]};
  const double h = cs[(c0 + 3) * cst];
  double p[3];
  panel_center(c, h, n, panel, p);
  W.p[3 * L.slot + 0] = p[0];
  W.p[3 * L.slot + 1] = p[1];
  W.p[3 * L.slot + 2] = p[2];
  W.rng[L.slot] = L.rng;
  // reductions, not load-add-store: nothing waits for the slot's counters
  atomicAdd(&W.mw[L.slot], 1u);
  atomicAdd(reinterpret_cast<unsigned long long*>(&W.mwsteps[L.slot]),
            static_cast<unsigned long long>(L.steps));
  W.state[L.slot] = S_ACTIVE;
}


struct DirDelta {
  uint64_t room;
  uint32_t node;
  uint32_t pad;
};

// interior steps (mw_step): words w with (w * 6 mod 2^32) >= kInteriorTie
// may straddle an f64 threshold and take the exact scan
constexpr uint32_t kInteriorTie = 0xFFFFFFFAu;

// One lattice step (microwalk.cpp:88-152) for lane L.  Every node takes the
// same code path: a neighbour inside the current cell has the node's own
// permittivity, so its alpha is e/(e+e) = 1/2 exactly; a neighbour across a
// cell face takes the face-neighbour class's alpha from the palette-pair
// table (1 on a lattice face).  The six alphas, their in-order partial sums
// and the scan are the reference's f64 arithmetic.  Returns 0 (moved inside
// the cell), 1 (surface exit through *xdir) or 2 (moved into the adjacent
// cell along *xdir; the caller refreshes the cell data).
template <int RNG>
__device__ __forceinline__ int mw_step(const DParams& P, const DirDelta* dd, MwLane& L, uint32_t w,
                                       uint64_t z, uint32_t tie_ctr, int* xdir) {
  ++L.steps;
  // exact zero-byte mask of the six room bytes: bit 8d+7 set <=> on face d
  const uint64_t r = L.room & 0x0000FFFFFFFFFFFFull;
  const uint64_t t = (r & 0x00007F7F7F7F7F7Full) + 0x00007F7F7F7F7F7Full;
  const uint64_t onface = ~(t | r | 0x00007F7F7F7F7F7Full) & 0x0000808080808080ull;
  if (RNG == FRW_RNG_PHILOX && onface == 0 && w * 6u < kInteriorTie) {
    // interior node: all six alphas are 1/2, so the scan below computes
    // sum = 3, acc_d = (d+1)/2 exactly and dir = #{d : (d+1)/2 <= fl(3x/2^53)}
    // for the 53-bit uniform x = w*2^21 + low21.  That count is floor(6w/2^32)
    // for every word w whose 2^21-wide interval contains none of the five
    // exact f64 thresholds; the words that can contain one have 6w within 6
    // of a multiple of 2^32 (the low word of w*6 >= kInteriorTie) and take
    // the scan (tests/test_step_law.py checks the equivalence exhaustively
    // around every threshold).
    const int dir = static_cast<int>(__umulhi(w, 6u));
    const DirDelta del = dd[dir];
    *xdir = dir;
    L.node += del.node;
    L.room += del.room;
    return 0;
  }
  double acc[6];
  double sum = 0;
#pragma unroll
  for (int d = 0; d < 6; ++d) {
    sum += ((onface >> (8 * d + 7)) & 1) ? L.al[d] : 0.5;
    acc[d] = sum;
  }
  if (onface) ++L.gsteps;
  int dir = 0;
  if (RNG == FRW_RNG_SPLITMIX_PARITY) {
    const double target = static_cast<double>(z >> 11) * 0x1.0p-53 * sum;
#pragma unroll
    for (int d = 0; d < 5; ++d) dir += acc[d] <= target;  // first d with target < acc_d
  } else {
    // the 32-bit word fixes x to [w*2^21, w*2^21 + 2^21): decide at both
    // ends; only when they disagree are the low 21 bits drawn
    const uint64_t xl = static_cast<uint64_t>(w) << 21;
    const double tl = static_cast<double>(xl) * 0x1.0p-53 * sum;
    const double th = static_cast<double>(xl | 0x1FFFFF) * 0x1.0p-53 * sum;
    int dh = 0;
#pragma unroll
    for (int d = 0; d < 5; ++d) {
      dir += acc[d] <= tl;
      dh += acc[d] <= th;
    }
    if (__builtin_expect(dh != dir, 0)) {
      const uint64_t x53 = xl | (philox53(P, L.wid, tie_ctr, 1u) & 0x1FFFFF);
      const double target = static_cast<double>(x53) * 0x1.0p-53 * sum;
      dir = 0;
#pragma unroll
      for (int d = 0; d < 5; ++d) dir += acc[d] <= target;
    }
  }
  const DirDelta del = dd[dir];
  *xdir = dir;
  if ((onface >> (8 * dir + 7)) & 1) {
    const int cn = static_cast<int>((L.fc >> (8 * dir)) & 0xFF);
    if (cn == kFace) return 1;  // left the lattice (microwalk.cpp:126-135)
    if (cn == kCond) return 3;  // absorbed by a conductor (microwalk.cpp:136-149)
    L.node += del.node;
    return 2;
  }
  L.node += del.node;
  L.room += del.room;
  return 0;
}

// alpha_sm: the palette-pair alphas, then alpha 1 (absorbing faces) at
// index P*P so a face alpha is one unconditional shared load (P <= PMAX)
__device__ AlphaTab setup_smem_tables(const DStruct& s, double* alpha_sm, DirDelta* dd,
                                      const DJump& Jg, JumpSmem& jsm, DJump* J) {
  // lattice-jump tables: every radius's meta, the alias tables of the radii
  // whose cumulative size fits kJumpSm
  *J = Jg;
  J->msm = 0;
  if (Jg.mmax >= 2) {
    int msm = 1;
    while (msm < Jg.mmax && Jg.meta[msm + 1].off + Jg.meta[msm + 1].K <= kJumpSm) ++msm;
    const int ne = msm >= 2 ? static_cast<int>(Jg.meta[msm].off + Jg.meta[msm].K) : 0;
    for (int i = threadIdx.x; i <= Jg.mmax; i += blockDim.x) jsm.meta[i] = Jg.meta[i];
    for (int i = threadIdx.x; i < ne; i += blockDim.x) {
      jsm.prob[i] = __ldg(Jg.prob + i);
      jsm.alias[i] = __ldg(Jg.alias + i);
    }
    J->msm = msm;
    J->meta = jsm.meta;
    J->prob_s = jsm.prob;
    J->alias_s = jsm.alias;
  }
  const bool small = s.P <= PMAX;
  if (small) {
    for (int i = threadIdx.x; i < s.P * s.P; i += blockDim.x) alpha_sm[i] = __ldg(s.alpha + i);
    if (threadIdx.x == 0) alpha_sm[s.P * s.P] = 1.0;
  }
  if (threadIdx.x < 6) {
    const int d = threadIdx.x, a = d >> 1;
    DirDelta x;
    // moving -a: distance to the low face -1, to the high face +1
    const uint64_t lo_b = 1ull << (16 * a), hi_b = 1ull << (16 * a + 8);
    x.room = (d & 1) ? (lo_b - hi_b) : (hi_b - lo_b);
    x.node = (d & 1) ? (1u << (8 * a)) : static_cast<uint32_t>(-(1 << (8 * a)));
    x.pad = 0;
    dd[d] = x;
  }
  __syncthreads();
  return AlphaTab{small ? alpha_sm : nullptr, s.pal, s.P, s.bg};
}

#ifndef FRW_STEP_UNROLL
#define FRW_STEP_UNROLL 0
#endif

// Events of a MicroWalk super-step
enum : int { MW_GO = 0, MW_SURFACE = 1, MW_COND = 3, MW_CAP = 4 };

// One lattice jump (see DJump) from 64 random bits when all six face
// distances are >= 2: radius m = min(face distances, mmax); the face is
// floor(6x), the position on it the CDF inversion of the fractional part;
// the walker moves to that node of the radius-m sphere (still in its cell),
// the face distances follow, and the hop's step count takes E[tau_m]
// (stochastically rounded).  Returns false (nothing consumed) otherwise.
// the jump of radius m (2 <= m <= mmax) from 64 random bits.  CHECK: the
// ball may reach beyond the lane's cell (a homogeneous-ball jump); a landing
// outside it leaves the cell pending (room 0, looked up next super-step)
template <bool CHECK = false>
__device__ __forceinline__ void mw_jump_r(const DJump& J, MwLane& L, int m, uint32_t w0,
                                          uint32_t w1) {
  const JumpMeta jm = J.meta[m];
  const uint64_t x = (static_cast<uint64_t>(w0) << 32) | w1;
  const int face = static_cast<int>(__umul64hi(x, 6ull));
  const uint64_t y = x * 6ull;  // uniform given the face
  // alias draw: column i uniform in [0, K), its fraction f uniform given i
  const uint32_t i = static_cast<uint32_t>(__umul64hi(y, jm.K));
  const uint64_t f = y * jm.K;
  const bool shared = m <= J.msm;
  const uint64_t thr = shared ? J.prob_s[jm.off + i] : __ldg(J.prob + jm.off + i);
  const uint32_t al = shared ? J.alias_s[jm.off + i] : __ldg(J.alias + jm.off + i);
  const uint32_t idx = f < thr ? i : al;
  const int side = static_cast<int>(jm.side);
  const int v = static_cast<int>(__umulhi(idx, jm.magic));
  const int u = static_cast<int>(idx) - v * side;
  const int a = face >> 1;
  // displacement: +-m along the face axis a, the panel's (u, v) across it in
  // the conventions of surface_panel_of (sgf.cpp:13-30: a=0 (y,z), a=1
  // (x,z), a=2 (x,y)); selects, not an indexed array (no local memory)
  const int sm = (face & 1) ? m : -m, du = u - (m - 1), dv = v - (m - 1);
  const int dl[3] = {a == 0 ? sm : du, a == 0 ? du : (a == 1 ? sm : dv), a == 2 ? sm : dv};
  L.node += static_cast<uint32_t>(dl[0] + dl[1] * 256 + dl[2] * 65536);
  // byte 2a: distance to the low face (+delta), byte 2a+1: to the high face
  long long dr = 0;
#pragma unroll
  for (int q = 0; q < 3; ++q)
    dr += static_cast<long long>(dl[q]) * ((1ll << (16 * q)) - (1ll << (16 * q + 8)));
  bool in_cell = true;
  if (CHECK) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int lo = static_cast<int>((L.room >> (16 * q)) & 0xFF);
      const int hi = static_cast<int>((L.room >> (16 * q + 8)) & 0xFF);
      in_cell &= dl[q] >= -lo && dl[q] <= hi;
    }
  }
  if (in_cell)
    L.room += static_cast<uint64_t>(dr);
  else
    L.room = 0;
  ++L.jumps;
  const int js = static_cast<int>(jm.esteps >> 32) +
                 (static_cast<uint32_t>(jm.esteps) > static_cast<uint32_t>(y >> 8) ? 1 : 0);
  L.steps += js;
  L.jsteps += js;
}

// The largest m such that every node within L-inf distance m of the lane's
// node lies in the lattice and in exactly the same clipped boxes (so has the
// same permittivity): each box either contains the whole ball or misses it.
// Inside that ball every alpha is 1/2 (microwalk.cpp:97-104), so the jump
// law of radius m holds there whatever cells the box faces cut (the cells are
// a tensor grid of every face, finer than the material boundaries).
// the largest m for which box b contains or misses the whole L-inf ball of
// radius m around node v
__device__ __forceinline__ int box_ball(uint64_t b, const int v[3]) {
  bool in = true;
  int gin = 64, gout = -1;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const int lo = box_lo(b, a), hi = box_hi(b, a);
    if (v[a] < lo) {
      in = false;
      gout = max(gout, lo - v[a] - 1);
    } else if (v[a] > hi) {
      in = false;
      gout = max(gout, v[a] - hi - 1);
    } else {
      gin = min(gin, min(v[a] - lo, hi - v[a]));
    }
  }
  return in ? gin : gout;
}
__device__ __forceinline__ int lattice_ball(const int v[3], int n) {
  int m = 31;
#pragma unroll
  for (int a = 0; a < 3; ++a) m = min(m, min(v[a], n - 1 - v[a]));
  return m;
}
// *hq: the box that brought the radius below 2 or set it (-1: the lattice)
__device__ int mw_hom_radius(const MwLane& L, int n, int* hq) {
  const int v[3] = {coord(L.node, 0), coord(L.node, 1), coord(L.node, 2)};
  int m = lattice_ball(v, n);
  int arg = -1;
#pragma unroll 1
  for (int q = 0; q < L.nbx && m >= 2; ++q) {
    const int mb = box_ball(L.bx[q], v);
    if (mb < m) {
      m = mb;
      arg = q;
    }
  }
  *hq = arg;
  return m;
}

__device__ __forceinline__ bool mw_jump(const DJump& J, MwLane& L, uint32_t w0, uint32_t w1) {
  const uint64_t r = L.room & 0x0000FFFFFFFFFFFFull;
  // bytes are < 128: byte | 0x80 minus 2 keeps its top bit iff byte >= 2
  if ((((r | 0x0000808080808080ull) - 0x0000020202020202ull) & 0x0000808080808080ull) !=
      0x0000808080808080ull)
    return false;
  int m = J.mmax;
#pragma unroll
  for (int d = 0; d < 6; ++d) m = min(m, static_cast<int>((r >> (8 * d)) & 0xFF));
  mw_jump_r(J, L, m, w0, w1);
  return true;
}

// Up to four lattice steps of the lane's hop from one Philox block (four
// SplitMix64 draws in parity mode); a move into another cell ends the
// super-step and refreshes the cell from the atlas.  Returns an MW_* event.
template <int RNG>
__device__ __forceinline__ int mw_superstep(const DParams& P, const DJump& J, const DSlots& W,
                                            const AlphaTab& AT, const DirDelta* dd, int n, int cap,
                                            MwLane& L, int* xdir) {
  uint32_t w4[4] = {0, 0, 0, 0};
  PH_T0(ph11);
  if (RNG == FRW_RNG_PHILOX) {
    const uint64_t id = P.walk_begin + L.wid;
    const U32x4 o = philox4x32_10(
        {static_cast<uint32_t>(id), static_cast<uint32_t>(id >> 32),
         static_cast<uint32_t>(L.rng), 2u},
        static_cast<uint32_t>(P.seed), static_cast<uint32_t>(P.seed >> 32));
    w4[0] = o.x;
    w4[1] = o.y;
    w4[2] = o.z;
    w4[3] = o.w;
  }
#ifdef FRW_PHASE_CLOCKS
  if (w4[0] == 0x12345678u) w4[1] ^= 1;  // keep the draw before the clock read
#endif
  PH_ADD(11, ph11);
  // a pending cell (new hop, or a move into another cell last super-step):
  // one inlined copy of the atlas lookup serves both
  PH_T0(ph5);
  if ((L.room >> 48) == 0) {
    PH_T0(ph4);
    mw_cell_change(AT, n, L);
    PH_ADD(4, ph4);
  }
  int code = 0;
  int u0 = 0;  // words taken by jumps (two per jump)
  PH_T0(ph12);
  if (RNG == FRW_RNG_PHILOX && J.mmax >= 2 && L.steps < cap) {
    if (mw_jump(J, L, w4[0], w4[1])) {
      u0 = 2;
      if (J.twice && L.steps < cap && mw_jump(J, L, w4[2], w4[3])) u0 = 4;
    } else if (J.hom) {
      // no room for a jump inside the cell: the homogeneous ball around the
      // node (a bound carried from the node it was computed at, recomputed
      // once it drops below 2)
      const int d = max(max(abs(coord(L.node, 0) - coord(L.hnode, 0)),
                            abs(coord(L.node, 1) - coord(L.hnode, 1))),
                        abs(coord(L.node, 2) - coord(L.hnode, 2)));
      // the radius is 1-Lipschitz in the node: within [hom - d, hom + d];
      // recompute only when that range straddles 2
      int eff = L.hom - d;
      if (eff < 2 && L.hom + d >= 2) {
        // the radius is at most what the box (or lattice) that limited it
        // last time allows here: the full O(boxes) scan only when that is >= 2
        const int v[3] = {coord(L.node, 0), coord(L.node, 1), coord(L.node, 2)};
        int lim = lattice_ball(v, n);
        if (L.hq >= 0) lim = min(lim, box_ball(L.bx[L.hq], v));
        if (lim >= 2) {
          PH_T0(ph14);
          int hq;
          eff = mw_hom_radius(L, n, &hq);
          L.hq = hq;
          PH_ADD(14, ph14);
          L.hom = eff;
          L.hnode = L.node;
        }
      }
      if (eff >= 2) {
        mw_jump_r<true>(J, L, min(eff, J.mmax), w4[0], w4[1]);
        u0 = (L.room >> 48) == 0 ? 4 : 2;  // left the cell: no steps before its lookup
      }
    }
  }
  PH_ADD(12, ph12);
  PH_T0(ph13);
#if FRW_STEP_UNROLL
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    if (u >= u0 && code == 0 && L.steps < cap) {
      uint64_t z = 0;
      if (RNG == FRW_RNG_SPLITMIX_PARITY) z = sm64_next(L.rng);
      code = mw_step<RNG>(P, dd, L, w4[u], z, static_cast<uint32_t>(L.rng * 4 + u), xdir);
    }
  }
#else
  // one copy of the step body (the unrolled four made the super-step ~24 KB
  // of SASS: warps stalled on instruction fetch at its reconvergence points)
#pragma unroll 1
  for (int u = u0; u < 4 && code == 0 && L.steps < cap; ++u) {
    const uint32_t w = u == 0 ? w4[0] : u == 1 ? w4[1] : u == 2 ? w4[2] : w4[3];
    uint64_t z = 0;
    if (RNG == FRW_RNG_SPLITMIX_PARITY) z = sm64_next(L.rng);
    code = mw_step<RNG>(P, dd, L, w, z, static_cast<uint32_t>(L.rng * 4 + u), xdir);
  }
#endif
  PH_ADD(13, ph13);
  if (RNG == FRW_RNG_PHILOX) ++L.rng;  // next 4-word block
  if (code == 2) {  // moved into another cell: looked up next super-step
    ++L.cchg;
    L.room = 0;
    code = 0;
  }
  PH_ADD(5, ph5);
  if (code == 0 && L.steps >= cap) return MW_CAP;
  return code;
}

// conductor exit: the walk terminates on the first declared conductor box
// holding the voxel across the face (engine.cpp:333-336 -> run_walk's
// Terminate branch)
__device__ void mw_conductor_exit(const DSlots& W, WalkRec* recs, DCounters* C, MwLane& L,
                                  int xdir) {
  int v[3] = {coord(L.node, 0), coord(L.node, 1), coord(L.node, 2)};
  v[xdir >> 1] += (xdir & 1) ? 1 : -1;
  const int ci = box_cond(L.bx[cond_box_at(L.bx, L.ncond, v)]);
  W.mw[L.slot] += 1;
  W.mwsteps[L.slot] += L.steps;
  finish_walk(W, recs, C, L.slot, ci, false);
}

__device__ __forceinline__ void flush_mw_stats_one(DCounters* C, const MwLane& L) {
  atomicAdd(&C->gen_steps, static_cast<unsigned long long>(L.gsteps));
  atomicAdd(&C->cell_chg, static_cast<unsigned long long>(L.cchg));
}

__device__ __forceinline__ void flush_mw_stats(DCounters* C, const MwLane& L) {
  unsigned long long g = L.gsteps, cc = L.cchg, jp = L.jumps, js = L.jsteps;
  for (int o = 16; o > 0; o >>= 1) {
    g += __shfl_xor_sync(0xFFFFFFFFu, g, o);
    cc += __shfl_xor_sync(0xFFFFFFFFu, cc, o);
    jp += __shfl_xor_sync(0xFFFFFFFFu, jp, o);
    js += __shfl_xor_sync(0xFFFFFFFFu, js, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&C->gen_steps, g);
    atomicAdd(&C->cell_chg, cc);
    atomicAdd(&C->jumps, jp);
    atomicAdd(&C->jsteps, js);
  }
}

// Cell-change batching: a lane whose hop moved into another cell looks the
// cell up at the start of its next super-step (cell_scan, O(boxes), ~1/5 of
// the lanes per pass).  With FRW_CC_NUM/FRW_CC_DEN > 0 such a lane sits out
// passes until that share of the warp's stepping lanes is waiting too (or one
// has waited FRW_CC_WAIT passes), so the lookup's instructions serve several
// lanes at once.  A waiting lane draws nothing: its stream position and
// hence its walk are unchanged.
#ifndef FRW_CC_NUM
#define FRW_CC_NUM 0
#endif
#ifndef FRW_CC_DEN
#define FRW_CC_DEN 1
#endif
#ifndef FRW_CC_WAIT
#define FRW_CC_WAIT 4
#endif
// stepping: the lane would run a super-step this pass; returns whether it
// should sit this pass out (all 32 lanes call)
__device__ __forceinline__ bool cc_hold(bool stepping, const MwLane& L, int& waited) {
#if FRW_CC_NUM > 0
  const bool pend = stepping && (L.room >> 48) == 0;
  const int np = __popc(__ballot_sync(0xFFFFFFFFu, pend));
  const int ns = __popc(__ballot_sync(0xFFFFFFFFu, stepping));
  const bool late = __any_sync(0xFFFFFFFFu, pend && waited >= FRW_CC_WAIT);
  const bool hold = pend && !late && np * FRW_CC_DEN < ns * FRW_CC_NUM;
  waited = hold ? waited + 1 : 0;
  return hold;
#else
  return false;
#endif
}

// persistent MicroWalk kernel: each thread runs queued hops back to back
#ifndef FRW_KMW_MINB
#define FRW_KMW_MINB 2  // 64 registers: two 512-thread CTAs per SM (+1-2% over one)
#endif
template <int RNG>
__global__ void __launch_bounds__(512, FRW_KMW_MINB)
    k_mw(DStruct s, DParams P, DSlots W, WalkRec* recs, DCounters* C, const int* queue,
         int* aq_out, int* mq_next) {
  __shared__ double alpha_sm[PMAX * PMAX + 1];  // used when P <= PMAX
  __shared__ DirDelta dd[6];
  extern __shared__ uint64_t frw_dsm[];  // kBoxSm box slices per thread (mw_arm)
  __shared__ JumpSmem jsm;
  DJump J;
  const AlphaTab AT = setup_smem_tables(s, alpha_sm, dd, P.jump, jsm, &J);
  const int n = P.n;
  const int cap = 1000 * n * n;  // microwalk.cpp:81
  const int slice = P.mw_slice > 0 ? P.mw_slice : 0x7FFFFFFF;
  const unsigned long long qlen = C->qlen;
  MwLane L;
  L.gsteps = 0;
  L.jumps = 0;
  L.jsteps = 0;
  L.cchg = 0;
  int left = slice;  // super-steps left in this visit of the hop
  // (popping one job ahead to take the queue read off the re-arm path lost
  // 3-8%: lanes holding a reserved job lengthen the round's last hops)
  auto pop = [&]() -> int {
    const unsigned long long it = atomicAdd(&C->qhead, 1ull);
    return it < qlen ? queue[it] : -1;
  };
  const int q0 = pop();
  bool live = q0 >= 0;
  if (live) {
    FRW_DCHECK(C, q0 >= 0 && q0 < W.S);
    mw_arm(W, q0, q0, n, L, frw_dsm);
  }
  int cc_waited = 0;
  while (__any_sync(0xFFFFFFFFu, live)) {
    int code = MW_GO, xdir = 0;
    const bool hold = cc_hold(live, L, cc_waited);
    if (live && !hold) {
      code = mw_superstep<RNG>(P, J, W, AT, dd, n, cap, L, &xdir);
      FRW_DCHECK(C, node_ok(L.node, n));
    }
    if (live && !hold && code == MW_GO && --left == 0) {
      mw_carry(W, C, mq_next, L);
      code = -1;
    }
    if (live && code != MW_GO) {
      if (code == MW_SURFACE) {
        mw_exit(W, n, L, xdir);
        mw_requeue(C, aq_out, L.slot);
      } else if (code == MW_COND) {
        mw_conductor_exit(W, recs, C, L, xdir);
      } else if (code != -1) {
        set_err(C, FRW_ESTEPCAP);
      }
      left = slice;
      const int q = pop();
      live = q >= 0;
      if (live) {
        FRW_DCHECK(C, q >= 0 && q < W.S);
        mw_arm(W, q, q, n, L, frw_dsm);
      }
    }
  }
  flush_mw_stats(C, L);
}

// ---- dense MicroWalk hops (more than KMAX boxes reach into the cube) -------
// The cell atlas holds at most KMAX boxes per cube.  Such a hop runs here:
// one CTA classifies every voxel centre of the cube against the structure
// (LazyField::classify, microwalk.cpp:44-71: conductor_at(p, 0) for the
// MicroWalk-E lattice, else permittivity_at -- the same closed-box tests
// the clipped boxes encode) into a u16 grid, and one lane walks the hop on
// it, every node a cell of its own (its six alphas from the palette pair,
// microwalk.cpp:97-104), with the walk's own random stream.  Rare by
// construction; the walk then rejoins the next round's ACTIVE queue.
constexpr uint16_t kDenseCondBit = 0x8000;
__device__ void dense_cell(const uint16_t* grid, const AlphaTab& T, int n, MwLane& L) {
  const int v[3] = {coord(L.node, 0), coord(L.node, 1), coord(L.node, 2)};
  const int g0 = grid[(v[2] * n + v[1]) * n + v[0]];
  uint64_t fc = 0;
#pragma unroll
  for (int d = 0; d < 6; ++d) {
    int w[3] = {v[0], v[1], v[2]};
    w[d >> 1] += (d & 1) ? 1 : -1;
    const bool out = w[d >> 1] < 0 || w[d >> 1] >= n;
    const int gn = out ? 0 : grid[(w[2] * n + w[1]) * n + w[0]];
    const bool cond = !out && (gn & kDenseCondBit);
    fc |= static_cast<uint64_t>(out ? kFace : (cond ? kCond : 0)) << (8 * d);
    if (out || cond)
      L.al[d] = 1.0;
    else if (T.tab)
      L.al[d] = T.tab[gn * T.Pn + g0];
    else {
      const double en = __ldg(T.pal + gn), e0 = __ldg(T.pal + g0);
      L.al[d] = en / (en + e0);
    }
  }
  L.fc = fc;
  L.room = 0x0101ull << 48;  // every node is a cell of its own: on all six faces
}

template <int RNG>
__global__ void __launch_bounds__(256)
    k_mw_dense(DStruct s, DParams P, DSlots W, WalkRec* recs, DCounters* C, const int* dense,
               int* aq_out, uint16_t* scratch) {
  __shared__ double alpha_sm[PMAX * PMAX + 1];  // used when P <= PMAX
  __shared__ DirDelta dd[6];
  __shared__ int job_sh;
  __shared__ JumpSmem jsm;
  DJump J;
  const AlphaTab AT = setup_smem_tables(s, alpha_sm, dd, P.jump, jsm, &J);
  const int n = P.n, nn = n * n, m3 = nn * n;
  const int cap = 1000 * n * n;
  uint16_t* grid = scratch + static_cast<size_t>(blockIdx.x) * m3;
  DParams Pd = P;
  Pd.jump.mmax = 0;  // no lattice jumps: a node's ball is not known to be homogeneous
  DJump Jd = J;
  Jd.mmax = 0;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned long long j = atomicAdd(&C->dqhead, 1ull);
      job_sh = j < C->dqlen ? dense[j] : -1;
    }
    __syncthreads();
    const int slot = job_sh;
    if (slot < 0) break;
    if (threadIdx.x == 0) atomicAdd(&C->dense_hops, 1ull);
    const double c[3] = {W.cube[4 * slot], W.cube[4 * slot + 1], W.cube[4 * slot + 2]};
    const double h = W.cube[4 * slot + 3];
    const double pitch = 2.0 * h / n;
    const bool with_cond = (W.mwkind[slot] & kDenseCond) != 0;
    for (int v = threadIdx.x; v < m3; v += blockDim.x) {
      const int i = v % n, j = (v / n) % n, k = v / nn;
      const double p[3] = {vcenter(c[0], h, pitch, i), vcenter(c[1], h, pitch, j),
                           vcenter(c[2], h, pitch, k)};
      const int ci = with_cond ? conductor_at(s, p, 0.0) : -1;
      grid[v] = ci >= 0 ? static_cast<uint16_t>(kDenseCondBit | ci)
                        : static_cast<uint16_t>(eps_class_at(s, p));
    }
    __syncthreads();
    if (threadIdx.x != 0) continue;
    MwLane L;
    L.gsteps = L.cchg = L.jumps = L.jsteps = 0;
    L.slot = L.jslot = slot;
    L.wid = W.wid[slot];
    const int mid = (n - 1) / 2;
    L.node = mid | (mid << 8) | (mid << 16);
    L.hnode = L.node;
    L.hom = 0;
    L.hq = -1;
    L.rng = W.rng[slot];
    L.ncond = L.nbx = 0;
    L.steps = 0;
    L.room = 0;
    int code = MW_GO, xdir = 0;
    while (code == MW_GO) {
      if ((L.room >> 48) == 0) dense_cell(grid, AT, n, L);
      code = mw_superstep<RNG>(Pd, Jd, W, AT, dd, n, cap, L, &xdir);
      FRW_DCHECK(C, node_ok(L.node, n));
    }
    if (code == MW_SURFACE) {
      mw_exit(W, n, L, xdir);
      mw_requeue(C, aq_out, slot);
    } else if (code == MW_COND) {
      int v[3] = {coord(L.node, 0), coord(L.node, 1), coord(L.node, 2)};
      v[xdir >> 1] += (xdir & 1) ? 1 : -1;
      const int ci = grid[(v[2] * n + v[1]) * n + v[0]] & ~kDenseCondBit;
      W.mw[slot] += 1;
      W.mwsteps[slot] += L.steps;
      finish_walk(W, recs, C, slot, ci, false);
    } else {
      set_err(C, FRW_ESTEPCAP);
      W.state[slot] = S_FREE;
    }
    flush_mw_stats_one(C, L);
  }
}

// Run-to-completion kernel for the tail of a run: once few walks remain,
// rounds would each cost the longest hop chain of the round, so every lane
// takes an ACTIVE walk and runs it to its end, alternating transitions and
// MicroWalk super-steps in-thread.  A table miss parks its walk as in
// k_advance (the host resolves misses once the other walks are done).
#ifndef FRW_TAIL_BLOCKS
#define FRW_TAIL_BLOCKS 2
#endif
constexpr int kTailBlocks = FRW_TAIL_BLOCKS;  // resident 256-thread CTAs per SM
#ifndef FRW_TAIL_CHAIN
#define FRW_TAIL_CHAIN 1  // transitions per k_tail iteration while cached
#endif
#ifndef FRW_TAIL_REPS
#define FRW_TAIL_REPS 32  // MicroWalk super-steps per transition in k_tail
#endif
#ifndef FRW_TAIL_VOTE
#define FRW_TAIL_VOTE 1  // phase vote (0: the fixed transition / MicroWalk alternation)
#endif
#ifndef FRW_TAIL_VOTE_T
#define FRW_TAIL_VOTE_T 1  // weights of the lanes waiting for a transition / inside a hop
#endif
#ifndef FRW_TAIL_VOTE_M
#define FRW_TAIL_VOTE_M 2  // (1:1 and 2:1 measured 1-2% behind 1:2 on C3-C5)
#endif
template <int RNG>
__global__ void __launch_bounds__(256, kTailBlocks)
    k_tail(DStruct s, DSgf T, DParams P, DSlots W, WalkRec* recs, DCounters* C, DMiss M,
           const int* aq, const int* mq) {
  __shared__ double alpha_sm[PMAX * PMAX + 1];  // used when P <= PMAX
  __shared__ DirDelta dd[6];
  extern __shared__ uint64_t frw_dsm[];  // kBoxSm box slices per thread (mw_arm)
  __shared__ JumpSmem jsm;
  DJump J;
  const AlphaTab AT = setup_smem_tables(s, alpha_sm, dd, P.jump, jsm, &J);
  const int n = P.n;
  const int cap = 1000 * n * n;
  // items: first the MicroWalk hops carried over from the last round (their
  // jobs in their slots' entries), then the ACTIVE walks
  const unsigned long long qc = C->qlen;
  const unsigned long long total = qc + C->alen;
  AdvLane A;
  MwLane L;
  L.gsteps = 0;
  L.jumps = 0;
  L.jsteps = 0;
  L.cchg = 0;
  bool in_mw = false;
  int arm_s = -1, arm_j = -1;  // a MicroWalk hop to arm (one inlined mw_arm: code size)
  const int jlane = W.jtail + blockIdx.x * blockDim.x + threadIdx.x;
  bool live = false;
  auto fetch = [&]() {
#ifdef FRW_TAIL_SOLO
    if (threadIdx.x & 31) {  // latency experiment: one walk per warp
      live = false;
      return;
    }
#endif
    const unsigned long long item = atomicAdd(&C->ahead, 1ull);
    live = item < total;
    if (!live) return;
    if (item < qc) {
      const int q = mq[item];
      FRW_DCHECK(C, q >= 0 && q < W.S);
      arm_s = arm_j = q;  // armed at the one mw_arm site below
      in_mw = true;
    } else {
      const int q = aq[item - qc];
      FRW_DCHECK(C, q >= 0 && q < W.S && jlane < W.J);
      adv_load(W, q, A);
      A.jslot = jlane;
      in_mw = false;
    }
  };
#ifdef FRW_PHASE_CLOCKS
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    atomicCAS(&g_tail_t0, 0ull, gtimer());
    g_in_tail = 1;
  }
#endif
  fetch();
  long long cyc_mw = 0, cyc_all = 0;  // warp-uniform clock64 spans
#if FRW_TAIL_VOTE
  // Phase vote: each pass the warp runs the phase more of its live lanes wait
  // for -- one transition each for the lanes between hops, or MicroWalk
  // super-steps for the lanes inside a hop, until the waiting lanes outnumber
  // them (ties alternate) -- instead of a fixed alternation, so either
  // phase's instructions run with at least half of the live lanes.
  bool last_adv = false;
  int cc_waited = 0;
  while (__any_sync(0xFFFFFFFFu, live)) {
    const long long c0 = clock64();
    if (arm_s >= 0) {
      mw_arm(W, arm_s, arm_j, n, L, frw_dsm);
      arm_s = -1;
    }
    const int nt = __popc(__ballot_sync(0xFFFFFFFFu, live && !in_mw));
    const int nm = __popc(__ballot_sync(0xFFFFFFFFu, live && in_mw));
    if (nt * FRW_TAIL_VOTE_T > nm * FRW_TAIL_VOTE_M || (nt * FRW_TAIL_VOTE_T == nm * FRW_TAIL_VOTE_M && !last_adv)) {
      last_adv = true;
      if (live && !in_mw) {
        const int r = advance_once<false, false>(s, T, P, W, recs, C, M, nullptr, A);
        if (r == 2) {
          in_mw = true;
          arm_s = A.slot;
          arm_j = A.jslot;
        } else if (r == 1) {
          fetch();
        }
      }
      cyc_all += clock64() - c0;
      continue;
    }
    last_adv = false;
    const long long c1 = clock64();
#pragma unroll 1
    for (int rep = 0; rep < FRW_TAIL_REPS; ++rep) {
      const int km = __popc(__ballot_sync(0xFFFFFFFFu, live && in_mw && arm_s < 0));
      const int kt = __popc(__ballot_sync(0xFFFFFFFFu, live && (!in_mw || arm_s >= 0)));
      if (km == 0 || km * FRW_TAIL_VOTE_M < kt * FRW_TAIL_VOTE_T) break;
      if (cc_hold(live && in_mw && arm_s < 0, L, cc_waited)) continue;
      if (!(live && in_mw) || arm_s >= 0) continue;
      int xdir = 0;
      const int code = mw_superstep<RNG>(P, J, W, AT, dd, n, cap, L, &xdir);
      FRW_DCHECK(C, node_ok(L.node, n));
      if (code == MW_GO) continue;
      in_mw = false;
      if (code == MW_SURFACE) {
        mw_exit(W, n, L, xdir);
        adv_load(W, L.slot, A);
        A.jslot = jlane;
        continue;
      }
      if (code == MW_COND)
        mw_conductor_exit(W, recs, C, L, xdir);
      else {
        set_err(C, FRW_ESTEPCAP);
        W.state[L.slot] = S_FREE;
      }
      fetch();
    }
    const long long c2 = clock64();
    cyc_mw += c2 - c1;
    cyc_all += c2 - c0;
  }
#else
  while (__any_sync(0xFFFFFFFFu, live)) {
    const long long c0 = clock64();
    if (live && !in_mw) {
      // up to FRW_TAIL_CHAIN transitions back to back while they are cached
      // hops (each would otherwise wait out a whole MicroWalk stretch)
      int r = advance_once<false, false>(s, T, P, W, recs, C, M, nullptr, A);
#pragma unroll 1
      for (int k = 1; k < FRW_TAIL_CHAIN && r == 0; ++k)
        r = advance_once<false, false>(s, T, P, W, recs, C, M, nullptr, A);
      if (r == 2) {
        in_mw = true;
        arm_s = A.slot;
        arm_j = A.jslot;
      } else if (r == 1) {
        fetch();
      }
    }
    if (arm_s >= 0) {
      mw_arm(W, arm_s, arm_j, n, L, frw_dsm);
      arm_s = -1;
    }
    // up to 32 super-steps per transition (a hop is ~50 super-steps): the
    // MicroWalk lanes run long stretches between the divergent transitions
    // (8: 1.64e7, 16: 1.76e7, 32: 1.76e7 C3 walks/s; C5 MWE best at 32)
    const long long c1 = clock64();
#pragma unroll 1
    for (int rep = 0; rep < FRW_TAIL_REPS; ++rep) {
      const unsigned mwm = __ballot_sync(0xFFFFFFFFu, live && in_mw && arm_s < 0);
      if (!mwm) break;
      if (!(live && in_mw) || arm_s >= 0) continue;  // (a hop fetched here is armed next iteration)
      int xdir = 0;
      const int code = mw_superstep<RNG>(P, J, W, AT, dd, n, cap, L, &xdir);
      FRW_DCHECK(C, node_ok(L.node, n));
      if (code == MW_GO) continue;
      in_mw = false;
      if (code == MW_SURFACE) {
        PH_T0(ph6);
        mw_exit(W, n, L, xdir);
        adv_load(W, L.slot, A);
        A.jslot = jlane;
        PH_ADD(6, ph6);
        continue;
      }
      if (code == MW_COND)
        mw_conductor_exit(W, recs, C, L, xdir);
      else {
        set_err(C, FRW_ESTEPCAP);
        W.state[L.slot] = S_FREE;
      }
      fetch();
    }
    const long long c2 = clock64();
    cyc_mw += c2 - c1;
    cyc_all += c2 - c0;
#ifdef FRW_PHASE_CLOCKS
    if (live || in_mw) {
      atomicAdd(&g_ph[PH_ROW + 9], static_cast<unsigned long long>(c1 - c0));
      atomicAdd(&g_ph[PH_ROW + 10], static_cast<unsigned long long>(c2 - c1));
      atomicAdd(&g_ph[PH_ROW + 25], 1ull);
    }
#endif
  }
#endif  // FRW_TAIL_VOTE
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&C->tail_mw_cyc, static_cast<unsigned long long>(cyc_mw));
    atomicAdd(&C->tail_all_cyc, static_cast<unsigned long long>(cyc_all));
  }

  flush_mw_stats(C, L);
}


// ---- warp-specialised run-to-completion kernel ----------------------------
// In k_tail one lane alternates transitions and MicroWalk stretches, so a
// cached hop (microseconds) waits out the warp's whole MicroWalk stretch and
// only ~7 of 32 lanes do useful work.  k_flow splits the roles by warp:
// advance warps take walks from the ACTIVE ring (first the round's ACTIVE
// list), run transitions until the walk needs a MicroWalk hop or ends, and
// push compiled jobs to the MicroWalk ring; MicroWalk warps run jobs back to
// back (lanes refilled independently, as in k_mw) and push surface exits to
// the ACTIVE ring.  Handoffs go through the slot arrays: the producer's
// writes are published by a gpu-scope fence before the ring entry, and the
// consumer fences after seeing the entry.  Every lane holds at most one ring
// reservation; the kernel ends when no walk is left in the flow (finished,
// parked by a table miss, or dropped by an error).
#ifndef FRW_FLOW_ADV_WARPS
#define FRW_FLOW_ADV_WARPS 3
#endif
#ifndef FRW_FLOW_SLEEP
#define FRW_FLOW_SLEEP 256  // ns between the ring polls of a warp with nothing in hand
#endif
constexpr int kFlowAdvWarps = FRW_FLOW_ADV_WARPS;  // of the 8 warps of a CTA

__device__ __forceinline__ int ring_poll(const int* ring, unsigned long long h, unsigned mask) {
  return *reinterpret_cast<const volatile int*>(ring + (h & mask));
}
__device__ __forceinline__ void ring_push(int* ring, unsigned long long* tail, unsigned mask,
                                          int slot) {
  __threadfence();  // the walk's slot data before its ring entry
  const unsigned long long t = atomicAdd(tail, 1ull);
  volatile int* e = ring + (t & mask);
  while (*e >= 0) __nanosleep(64);  // (a wrapped entry not yet consumed)
  *e = slot;
}
__device__ __forceinline__ unsigned long long flow_live(const DCounters* C) {
  return *reinterpret_cast<const volatile unsigned long long*>(&C->flive);
}

__global__ void k_flow_init(DCounters* C) {
  C->fah = C->fat = C->fmh = C->fmt = 0;
  C->flive = C->alen + C->qlen;  // ACTIVE walks and the hops carried over from the last round
}

// Roles by SM instead of by warp (DParams::flow_adv of the flow_sms SM pairs
// run transitions, the others MicroWalk hops): an SM then fetches only its
// role's code -- k_tail's top stall is instruction fetch, its transition and
// MicroWalk paths together are three times the 32 KB L1.5 instruction cache.

// this SM's role: flow_adv of the flow_sms SM pairs run transitions, evenly
// spread (SM ids 2t and 2t+1, one TPC, share a role: measured, mixed pairs
// lose the instruction-cache benefit)
__device__ __forceinline__ bool flow_sm_adv(const DParams& P) {
  unsigned smid;
  asm("mov.u32 %0, %%smid;" : "=r"(smid));
  const unsigned m = (smid >> 1) % static_cast<unsigned>(P.flow_sms);
  return (m + 1) * P.flow_adv / P.flow_sms != m * P.flow_adv / P.flow_sms;
}

// the transition role: walks from the round's ACTIVE list, then from the
// ACTIVE ring; one transition per pass until the walk needs a MicroWalk hop
// (compiled here, pushed to the MicroWalk ring) or ends
__device__ __forceinline__ void flow_adv_loop(const DStruct& s, const DSgf& T, const DParams& P,
                                              const DSlots& W, WalkRec* recs, DCounters* C,
                                              const DMiss& M, const int* aq, int* ring_a,
                                              int* ring_m, unsigned mask) {
  const unsigned long long alen = C->alen;
  long long cyc_busy = 0;  // warp-uniform clock64 spans with work in hand
  AdvLane A;
  bool have = false, first = true;
  long long res = -1;  // reserved ACTIVE-ring index
  for (;;) {
    if (!have) {
      if (first) {
        const unsigned long long item = atomicAdd(&C->ahead, 1ull);
        if (item < alen) {
          FRW_DCHECK(C, aq[item] >= 0 && aq[item] < W.S);
          adv_load(W, aq[item], A);
          have = true;
        } else {
          first = false;
        }
      }
      if (!have && !first) {
        if (res < 0) res = static_cast<long long>(atomicAdd(&C->fah, 1ull));
        const int v = ring_poll(ring_a, res, mask);
        if (v >= 0) {
          FRW_DCHECK(C, v < W.S);
          ring_a[res & mask] = -1;
          __threadfence();
          FRW_DCHECK(C, W.state[v] == S_ACTIVE);  // (after the fence: the producer's writes are visible)
          adv_load(W, v, A);
          have = true;
          res = -1;
        }
      }
    }
    if (!__any_sync(0xFFFFFFFFu, have)) {
      if (flow_live(C) == 0) break;
      __nanosleep(FRW_FLOW_SLEEP);
      continue;
    }
    const long long c0 = clock64();
    if (have) {
      const int r = advance_once<false, false>(s, T, P, W, recs, C, M, nullptr, A);
      if (r == 2) {
        ring_push(ring_m, &C->fmt, mask, A.slot);
        have = false;
      } else if (r == 1) {
        atomicAdd(&C->flive, ~0ull);  // -1
        have = false;
      }
    }
    cyc_busy += clock64() - c0;
  }
  // T_MW: the busy cycles of the MicroWalk warps over those of all warps
  if ((threadIdx.x & 31) == 0)
    atomicAdd(&C->tail_all_cyc, static_cast<unsigned long long>(cyc_busy));
}

#ifndef FRW_FLOW_POLL
#define FRW_FLOW_POLL 4
#endif
// the MicroWalk role: the hops carried over from the last round, then jobs
// from the MicroWalk ring, back to back (lanes refilled independently, as in
// k_mw); surface exits go to the ACTIVE ring
template <int RNG>
__device__ __forceinline__ void flow_mw_loop(const DParams& P, const DJump& J, const DSlots& W,
                                             const AlphaTab& AT, const DirDelta* dd,
                                             WalkRec* recs, DCounters* C, const int* mq,
                                             int* ring_a, int* ring_m, unsigned mask,
                                             uint64_t* bsm) {
  const int n = P.n;
  const unsigned long long qlen = C->qlen;
  long long cyc_busy = 0;
  const int cap = 1000 * n * n;  // microwalk.cpp:81
  MwLane L;
  L.gsteps = 0;
  L.jumps = 0;
  L.jsteps = 0;
  L.cchg = 0;
  bool have = false, firstm = qlen > 0;
  long long res = -1;
  // a warp with hops in hand lets its idle lanes look for a job only every
  // FRW_FLOW_POLL-th pass: the ring poll is a dependent L2 round trip that the
  // stepping lanes of the warp would wait out on every super-step
  unsigned pass = 0;
  bool busy = false;
  for (;;) {
    const bool look = !busy || (pass++ % FRW_FLOW_POLL) == 0;
    if (!have && firstm && look) {  // the hops carried over from the last round first
      const unsigned long long item = atomicAdd(&C->qhead, 1ull);
      if (item < qlen) {
        const int q = mq[item];
        FRW_DCHECK(C, q >= 0 && q < W.S);
        mw_arm(W, q, q, n, L, bsm);
        have = true;
      } else {
        firstm = false;
      }
    }
    if (!have && !firstm && look) {
      if (res < 0) res = static_cast<long long>(atomicAdd(&C->fmh, 1ull));
      const int v = ring_poll(ring_m, res, mask);
      if (v >= 0) {
        FRW_DCHECK(C, v < W.S);
        ring_m[res & mask] = -1;
        __threadfence();
        mw_arm(W, v, v, n, L, bsm);
        have = true;
        res = -1;
      }
    }
    busy = __any_sync(0xFFFFFFFFu, have);
    if (!busy) {
      if (flow_live(C) == 0) break;
      __nanosleep(FRW_FLOW_SLEEP);
      continue;
    }
    const long long c0 = clock64();
    if (have) {
      int xdir = 0;
      const int code = mw_superstep<RNG>(P, J, W, AT, dd, n, cap, L, &xdir);
      FRW_DCHECK(C, node_ok(L.node, n));
      if (code != MW_GO) {
        have = false;
        if (code == MW_SURFACE) {
          mw_exit(W, n, L, xdir);
          ring_push(ring_a, &C->fat, mask, L.slot);
        } else {
          if (code == MW_COND)
            mw_conductor_exit(W, recs, C, L, xdir);
          else {
            set_err(C, FRW_ESTEPCAP);
            W.state[L.slot] = S_FREE;
          }
          atomicAdd(&C->flive, ~0ull);  // -1
        }
      }
    }
    cyc_busy += clock64() - c0;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&C->tail_mw_cyc, static_cast<unsigned long long>(cyc_busy));
    atomicAdd(&C->tail_all_cyc, static_cast<unsigned long long>(cyc_busy));
  }
  flush_mw_stats(C, L);
}

// one kernel, both roles: by SM pair (P.flow_sms > 0) or by warp
template <int RNG>
__global__ void __launch_bounds__(256, kTailBlocks)
    k_flow(DStruct s, DSgf T, DParams P, DSlots W, WalkRec* recs, DCounters* C, DMiss M,
           const int* aq, const int* mq, int* ring_a, int* ring_m, unsigned mask) {
  __shared__ double alpha_sm[PMAX * PMAX + 1];  // used when P <= PMAX
  __shared__ DirDelta dd[6];
  extern __shared__ uint64_t frw_dsm[];  // kBoxSm box slices per thread (mw_arm)
  __shared__ JumpSmem jsm;
  DJump J;
  const AlphaTab AT = setup_smem_tables(s, alpha_sm, dd, P.jump, jsm, &J);
  const bool adv_role = P.flow_sms > 0 ? flow_sm_adv(P) : (threadIdx.x >> 5) < kFlowAdvWarps;
  if (adv_role)
    flow_adv_loop(s, T, P, W, recs, C, M, aq, ring_a, ring_m, mask);
  else
    flow_mw_loop<RNG>(P, J, W, AT, dd, recs, C, mq, ring_a, ring_m, mask, frw_dsm);
}

// The two roles as two kernels, launched side by side on two streams, each
// with the registers and shared memory of its role (the transition kernel as
// k_advance: 4 x 256 threads per SM and no tables; the MicroWalk kernel as
// k_mw: 2 x 512 threads per SM at 64 registers with the jump tables and box
// slices).  A CTA that lands on an SM of the other role exits at once, so each
// SM fills up with CTAs of its own role; CTAs left over once their SMs are
// full run (and exit) when the flow has ended.
#ifndef FRW_FLOWADV_MINB
#define FRW_FLOWADV_MINB 4
#endif
__global__ void __launch_bounds__(256, FRW_FLOWADV_MINB)
    k_flow_adv(DStruct s, DSgf T, DParams P, DSlots W, WalkRec* recs, DCounters* C, DMiss M,
               const int* aq, int* ring_a, int* ring_m, unsigned mask) {
  if (!flow_sm_adv(P) || flow_live(C) == 0) return;
  flow_adv_loop(s, T, P, W, recs, C, M, aq, ring_a, ring_m, mask);
}

template <int RNG>
__global__ void __launch_bounds__(512, 2)
    k_flow_mw(DStruct s, DParams P, DSlots W, WalkRec* recs, DCounters* C, const int* mq,
              int* ring_a, int* ring_m, unsigned mask) {
  if (flow_sm_adv(P) || flow_live(C) == 0) return;
  __shared__ double alpha_sm[PMAX * PMAX + 1];  // used when P <= PMAX
  __shared__ DirDelta dd[6];
  extern __shared__ uint64_t frw_dsm[];  // kBoxSm box slices per thread (mw_arm)
  __shared__ JumpSmem jsm;
  DJump J;
  const AlphaTab AT = setup_smem_tables(s, alpha_sm, dd, P.jump, jsm, &J);
  flow_mw_loop<RNG>(P, J, W, AT, dd, recs, C, mq, ring_a, ring_m, mask, frw_dsm);
}

// ---- single transits over structure cubes (the single-transit API) --------
// microwalk_transit_lazy / microwalk_e_transit (microwalk.cpp:199-228): one
// thread per transit compiles the cube into slot t and walks it with the
// caller's SplitMix64 state (the lane machinery of k_mw in parity mode).
struct DevExit {
  int32_t kind, panel, conductor, dir;
  int32_t voxel[3];
  int32_t steps;
  double point[3];
};
static_assert(sizeof(DevExit) == sizeof(frw_exit), "exit layout");

// RNG = PHILOX: transit t draws from Philox (seed, t) (states unused) and
// takes lattice jumps when P.jump is set -- the production-mode transit law
template <int RNG>
__global__ void __launch_bounds__(128)
    k_transits(DStruct s, DParams P, DSlots W, DCounters* C, const double* cubes,
               const uint64_t* states, int count, int with_cond, int cap, DevExit* out) {
  __shared__ double alpha_sm[PMAX * PMAX + 1];  // used when P <= PMAX
  __shared__ DirDelta dd[6];
  __shared__ JumpSmem jsm;
  DJump J;
  const AlphaTab AT = setup_smem_tables(s, alpha_sm, dd, P.jump, jsm, &J);
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  const int n = P.n;
  const double c[3] = {cubes[4 * t], cubes[4 * t + 1], cubes[4 * t + 2]};
  const double h = cubes[4 * t + 3];
  DevExit e{};
  e.conductor = -1;
  e.panel = -1;
  const int rc = compile_mw_job(s, W, t, c, h, n, with_cond != 0, false, C);
  if (rc != 1) {
    if (rc == 3) set_err(C, FRW_EINVAL);  // the single-transit API keeps the KMAX cap
    e.kind = rc == 0 ? -1 : -2;  // EngulfedStart / too many boxes (error set)
    out[t] = e;
    return;
  }
  W.wid[t] = t;
  W.rng[t] = RNG == FRW_RNG_PHILOX ? 0 : states[t];
  W.mw[t] = 0;
  W.mwsteps[t] = 0;
  MwLane L;
  L.gsteps = 0;
  L.jumps = 0;
  L.jsteps = 0;
  L.cchg = 0;
  mw_arm(W, t, t, n, L, nullptr);
  int code = MW_GO, xdir = 0;
  while (code == MW_GO)
    code = mw_superstep<RNG>(P, J, W, AT, dd, n, cap, L, &xdir);
  const int a = xdir >> 1;
  e.kind = code == MW_SURFACE ? 0 : 1;
  e.dir = xdir;
  e.steps = L.steps;
  e.voxel[0] = coord(L.node, 0);
  e.voxel[1] = coord(L.node, 1);
  e.voxel[2] = coord(L.node, 2);
  if (code == MW_SURFACE) {
    const int u = a == 0 ? e.voxel[1] : e.voxel[0];
    const int v = a == 2 ? e.voxel[1] : e.voxel[2];
    e.panel = (xdir * n + v) * n + u;  // surface_panel_of (sgf.cpp:13-30)
    panel_center(c, h, n, e.panel, e.point);
  } else if (code == MW_COND) {
    int v[3] = {e.voxel[0], e.voxel[1], e.voxel[2]};
    v[a] += (xdir & 1) ? 1 : -1;
    e.conductor = box_cond(L.bx[cond_box_at(L.bx, L.ncond, v)]);
    // lattice_voxel_center + half a pitch towards the conductor
    // (microwalk.cpp:24-30, :141-143)
    const double pitch = 2.0 * h / n;
#pragma unroll
    for (int q = 0; q < 3; ++q) e.point[q] = vcenter(c[q], h, pitch, e.voxel[q]);
    e.point[a] += ((xdir & 1) ? 1 : -1) * h / n;
  } else {
    e.kind = -3;
    set_err(C, FRW_ESTEPCAP);
  }
  out[t] = e;
}

// ---- single engine transitions (Engine::first_transition / transition) -----
struct DevFirst {
  int32_t ok, branch;
  double weight;
  double point[3];
};
static_assert(sizeof(DevFirst) == sizeof(frw_first), "first layout");
struct DevEvent {
  int32_t kind, conductor, dispatch, pad;
  double point[3];
  uint64_t mw_steps;
};
static_assert(sizeof(DevEvent) == sizeof(frw_event), "event layout");

// rc per entry: 1 done, 2 table miss (re-run after the key is inserted), <0 error
__global__ void __launch_bounds__(128)
    k_first_single(DStruct s, DSgf T, DParams P, DSlots W, DCounters* C, DMiss M,
                   const double* gpts, const int32_t* axsign, uint64_t* states, const int* idx,
                   int count, int* rc_out, DevFirst* out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= count) return;
  const int t = idx[q];
  Rng rng;
  rng.s = states[t];
  const double g[3] = {gpts[3 * t], gpts[3 * t + 1], gpts[3 * t + 2]};
  FirstOut fo;
  const int rc = first_transition(s, T, P, t, rng, g, axsign[2 * t], axsign[2 * t + 1],
                                  W.boxes + static_cast<size_t>(q) * KMAX, C, M, &fo);
  rc_out[q] = rc;
  if (rc == 2) return;  // miss: nothing drawn, the state stays
  DevFirst f{};
  f.ok = rc == 1;
  if (rc == 1) {
    f.branch = fo.branch;
    f.weight = fo.weight;
    f.point[0] = fo.p[0];
    f.point[1] = fo.p[1];
    f.point[2] = fo.p[2];
  }
  out[t] = f;
  states[t] = rng.s;
  if (rc < 0) set_err(C, FRW_EINVAL);
}

__global__ void __launch_bounds__(128)
    k_transition_single(DStruct s, DSgf T, DParams P, DSlots W, WalkRec* recs, DCounters* C,
                        DMiss M, const double* pts, uint64_t* states, const int* idx, int count,
                        int* rc_out, DevEvent* out) {
  __shared__ double alpha_sm[PMAX * PMAX + 1];  // used when P <= PMAX
  __shared__ DirDelta dd[6];
  __shared__ JumpSmem jsm;
  DJump J;
  const AlphaTab AT = setup_smem_tables(s, alpha_sm, dd, P.jump, jsm, &J);
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= count) return;
  const int t = idx[q];
  const int slot = q;
  W.wid[slot] = t;
  W.p[3 * slot] = pts[3 * t];
  W.p[3 * slot + 1] = pts[3 * t + 1];
  W.p[3 * slot + 2] = pts[3 * t + 2];
  W.rng[slot] = states[t];
  W.hops[slot] = 0;
  W.cached[slot] = 0;
  W.mw[slot] = 0;
  W.mwsteps[slot] = 0;
  W.weight[slot] = 0;
  W.state[slot] = S_ACTIVE;
  recs[t].done = 0;
  AdvLane L;
  adv_load(W, slot, L);
  const int r = advance_once(s, T, P, W, recs, C, M, nullptr, L);
  DevEvent e{};
  e.conductor = -1;
  e.dispatch = -1;
  if (r == 0) {  // cached hop
    e.kind = 0;
    e.dispatch = 0;
    e.point[0] = L.p[0];
    e.point[1] = L.p[1];
    e.point[2] = L.p[2];
    states[t] = L.rng.s;
  } else if (r == 1) {
    if (W.state[slot] == S_NEED_MW && (W.mwkind[slot] & kDense)) {
      set_err(C, FRW_EINVAL);  // the single-transition API keeps the KMAX cap
      rc_out[q] = 2;
      return;
    }
    if (!recs[t].done) {  // table miss (or geometry error, flagged in C->err)
      rc_out[q] = 2;
      return;
    }
    const int sl = recs[t].slot;
    e.kind = sl == s.nc ? 2 : 1;
    e.conductor = sl == s.nc ? -1 : sl;
    states[t] = L.rng.s;
  } else if (W.mwkind[slot] == 2) {  // FDM: solved by k_fdm, events gathered after
    rc_out[q] = 3;
    return;
  } else {  // MicroWalk / MicroWalk-E hop on the compiled job
    const int n = P.n;
    const int cap = 1000 * n * n;
    MwLane ml;
    ml.gsteps = 0;
    ml.jumps = 0;
    ml.jsteps = 0;
    ml.cchg = 0;
    mw_arm(W, slot, slot, n, ml, nullptr);
    ml.wid = t;
    int code = MW_GO, xdir = 0;
    while (code == MW_GO)
      code = mw_superstep<FRW_RNG_SPLITMIX_PARITY>(P, J, W, AT, dd, n, cap, ml, &xdir);
    e.dispatch = W.mwkind[slot] ? 2 : 1;
    e.mw_steps = ml.steps;
    if (code == MW_SURFACE) {
      mw_exit(W, n, ml, xdir);
      e.kind = 0;
      e.point[0] = W.p[3 * slot];
      e.point[1] = W.p[3 * slot + 1];
      e.point[2] = W.p[3 * slot + 2];
    } else if (code == MW_COND) {
      int v[3] = {coord(ml.node, 0), coord(ml.node, 1), coord(ml.node, 2)};
      v[xdir >> 1] += (xdir & 1) ? 1 : -1;
      e.kind = 1;
      e.conductor = box_cond(ml.bx[cond_box_at(ml.bx, ml.ncond, v)]);
    } else {
      set_err(C, FRW_ESTEPCAP);
    }
    states[t] = ml.rng;
  }
  rc_out[q] = 1;
  out[t] = e;
}

// ---- FDM transitions (engine.cpp:311-318) ------------------------------------
// One CTA per general cube: the voxel classes come from the job's cell atlas
// (the same voxelisation as build_grid, geometry.cpp:320-349); s_ii of the FD
// system (sgf.cpp:57-155) is applied matrix-free from palette-pair tables;
// Jacobi-PCG from zero to |r| < 1e-10 |b| (cap 20 rows) gives the adjoint row
// of the start node, probs = A_IB^T (eps .* z) with the normalisation check of
// sgf.cpp:249-253; the CDF is summed in panel order and sampled with one
// uniform (upper_bound, sgf.cpp:301-308).
constexpr int kFdmThreads = 1024;

__device__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < static_cast<int>(blockDim.x >> 5) ? red[l] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if (l == 0) red[32] = v;
  }
  __syncthreads();
  return red[32];
}
constexpr int kFdmMaxN = 32;  // voxel classes held in shared memory
constexpr int kFdmClasses = KMAX + 1;  // job-local classes (class_of)
struct FdmQueue {
  const int* queue;
  const unsigned long long* qlen;
  unsigned long long* qhead;
  int* out;                     // next-round ACTIVE queue (null: none)
  unsigned long long* outlen;
};

__device__ __forceinline__ void fdm_row(const uint8_t* cls, const double* pal, const double* apair,
                                        const double* spair, int Pn, int n, int v, double* diag,
                                        double off[6], int nbr[6]) {
  const int nn = n * n;
  const int c[3] = {v % n, (v / n) % n, v / nn};
  const int cv = cls[v];
  double rs = 0;
#pragma unroll
  for (int d = 0; d < 6; ++d) {
    const int a = d >> 1;
    const int st = a == 0 ? 1 : (a == 1 ? n : nn);
    const bool face = (d & 1) ? c[a] == n - 1 : c[a] == 0;
    if (face) {  // cube-surface panel: alpha 1, no interior coupling
      rs += 1.0;
      off[d] = 0.0;
      nbr[d] = v;
      continue;
    }
    const int u = (d & 1) ? v + st : v - st;
    const int q = cls[u] * Pn + cv;
    rs += apair[q];
    off[d] = spair[q];
    nbr[d] = u;
  }
  *diag = pal[cv] * rs;
}

__device__ __forceinline__ double2 block_sum2(double a, double b, double* red) {
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xFFFFFFFFu, a, o);
    b += __shfl_xor_sync(0xFFFFFFFFu, b, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) {
    red[w] = a;
    red[32 + w] = b;
  }
  __syncthreads();
  if (w == 0) {
    a = l < static_cast<int>(blockDim.x >> 5) ? red[l] : 0.0;
    b = l < static_cast<int>(blockDim.x >> 5) ? red[32 + l] : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xFFFFFFFFu, a, o);
      b += __shfl_xor_sync(0xFFFFFFFFu, b, o);
    }
    if (l == 0) {
      red[64] = a;
      red[65] = b;
    }
  }
  __syncthreads();
  return make_double2(red[64], red[65]);
}

// PSM: the search direction p lives in shared memory (the SpMV reads six
// neighbours of every node from it); the other Krylov vectors stay in the
// CTA's L2-resident scratch slab.
template <bool PSM>
__global__ void __launch_bounds__(kFdmThreads)
    k_fdm(DStruct s, DParams P, DSlots W, DCounters* C, FdmQueue Q, double* slab) {
  extern __shared__ __align__(16) uint8_t fsm[];
  __shared__ double red[66];
  __shared__ int job_sh;
  // voxel classes are job-local (class_of): the job's permittivities and
  // their pair tables are rebuilt per job, Pn = KMAX + 1 local classes
  const int n = P.n, m = n * n * n, nn = n * n, Pn = kFdmClasses;
  const int panels = 6 * nn;
  double* pal = reinterpret_cast<double*>(fsm);
  double* apair = pal + Pn;
  double* spair = apair + Pn * Pn;
  double* psm = spair + Pn * Pn;  // [m] when PSM
  uint8_t* cls = reinterpret_cast<uint8_t*>(PSM ? psm + m : psm);
  double* x = slab + static_cast<size_t>(blockIdx.x) * 5 * m;
  double* r = x + m;
  double* p = PSM ? psm : r + m;
  double* t = r + 2 * m;
  double* dinv = t + m;
  const int cc = (n - 1) / 2;
  const int crow = (cc * n + cc) * n + cc;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned long long j = atomicAdd(Q.qhead, 1ull);
      job_sh = j < *Q.qlen ? static_cast<int>(j) : -1;
    }
    __syncthreads();
    const int job = job_sh;
    if (job < 0) break;
    const int slot = Q.queue[job];
    // voxel classes of the cube from the job's atlas
    const uint64_t* A = lane_atlas(W, slot);
    const uint64_t bm[3] = {A[kAtBm], A[kAtBm + 1], A[kAtBm + 2]};
    const uint64_t cm = cond_mask(W.nbox[slot] & 0xFF);
    for (int v = threadIdx.x; v < m; v += blockDim.x) {
      const int vv[3] = {v % n, (v / n) % n, v / nn};
      cls[v] = static_cast<uint8_t>(class_of(voxel_mask(A, bm, vv), cm));
    }
    // (entries of local classes the job does not use are never read)
    for (int i = threadIdx.x; i < Pn; i += blockDim.x) {
      const int g = global_class(A, i, s.bg);
      pal[i] = g < s.P ? __ldg(s.pal + g) : 1.0;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < Pn * Pn; q += blockDim.x) {
      const double ei = pal[q / Pn], ev = pal[q % Pn];
      apair[q] = ei / (ei + ev);          // sgf.cpp:129
      spair[q] = -(ev * ei) / (ev + ei);  // sgf.cpp:135-137, bit-symmetric
    }
    __syncthreads();
    // PCG on s_ii z = e_c (Jacobi preconditioner, x0 = 0)
    double rz_loc = 0;
    for (int v = threadIdx.x; v < m; v += blockDim.x) {
      double dg, off[6];
      int nb[6];
      fdm_row(cls, pal, apair, spair, Pn, n, v, &dg, off, nb);
      const double b = v == crow ? 1.0 : 0.0;
      const double di = 1.0 / dg;
      dinv[v] = di;
      x[v] = 0.0;
      r[v] = b;
      p[v] = b * di;
      rz_loc += b * (b * di);
    }
    const double thresh = 1e-20;  // (rel_tol 1e-10)^2 |e_c|^2
    double rz = block_sum(rz_loc, red);
    double res2 = 1.0;
    const long cap = 20L * m;
    long it = 0;
    while (res2 >= thresh && it < cap) {
      double pt = 0;
      for (int v = threadIdx.x; v < m; v += blockDim.x) {
        double dg, off[6];
        int nb[6];
        fdm_row(cls, pal, apair, spair, Pn, n, v, &dg, off, nb);
        double acc = dg * p[v];
#pragma unroll
        for (int d = 0; d < 6; ++d) acc += off[d] * p[nb[d]];
        t[v] = acc;
        pt += p[v] * acc;
      }
      const double alpha = rz / block_sum(pt, red);
      double rr = 0, rzn = 0;
      for (int v = threadIdx.x; v < m; v += blockDim.x) {
        x[v] += alpha * p[v];
        const double rv = r[v] - alpha * t[v];
        r[v] = rv;
        rr += rv * rv;
        rzn += rv * (rv * dinv[v]);
      }
      const double2 sums = block_sum2(rr, rzn, red);
      res2 = sums.x;
      const double rz_new = sums.y;
      ++it;
      if (res2 < thresh) break;
      const double beta = rz_new / rz;
      rz = rz_new;
      for (int v = threadIdx.x; v < m; v += blockDim.x) p[v] = r[v] * dinv[v] + beta * p[v];
      __syncthreads();
    }
    // probs = A_IB^T (eps .* z), panel = (face*n + w)*n + u (sgf.hpp:34-36)
    double sum_loc = 0;
    for (int q = threadIdx.x; q < panels; q += blockDim.x) {
      const int face = q / nn, rem = q - face * nn;
      const int u = rem % n, w = rem / n;
      const int a = face >> 1;
      int ci[3];
      ci[a] = (face & 1) ? n - 1 : 0;
      ci[a == 0 ? 1 : 0] = u;
      ci[a == 2 ? 1 : 2] = w;
      const int v = (ci[2] * n + ci[1]) * n + ci[0];
      const double pr = pal[cls[v]] * x[v];
      t[q] = pr;
      sum_loc += pr;
    }
    const double psum = block_sum(sum_loc, red);
    __syncthreads();
    if (threadIdx.x == 0) {
      bool bad = res2 >= thresh || fabs(psum - 1.0) > 1e-9;
      // sequential CDF in panel order (sgf.cpp:255-262), min check
      double run = 0;
      for (int q = 0; q < panels; ++q) {
        const double pr = t[q];
        bad |= pr < -1e-9;
        run += pr > 0.0 ? pr : 0.0;
        t[q] = run;
      }
      if (bad) {
        set_err(C, FRW_ESOLVE);
        W.state[slot] = S_FREE;
      } else {
        Rng rng;
        rng.s = W.rng[slot];
        const long long wid = W.wid[slot];
        const double target = uniform(P, wid, rng) * run;
        int lo = 0, hi = panels;  // upper_bound
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (t[mid] <= target)
            lo = mid + 1;
          else
            hi = mid;
        }
        const int panel = lo == panels ? panels - 1 : lo;
        const double c[3] = {W.cube[4 * slot], W.cube[4 * slot + 1], W.cube[4 * slot + 2]};
        double pt3[3];
        panel_center(c, W.cube[4 * slot + 3], n, panel, pt3);
        W.p[3 * slot] = pt3[0];
        W.p[3 * slot + 1] = pt3[1];
        W.p[3 * slot + 2] = pt3[2];
        W.rng[slot] = rng.s;
        W.mw[slot] += 1;
        W.state[slot] = S_ACTIVE;
        if (Q.out) Q.out[atomicAdd(Q.outlen, 1ull)] = slot;
      }
    }
  }
}

// events of single FDM transitions solved by k_fdm (slot q holds entry idx[q])
__global__ void k_fdm_events(DSlots W, const int* slots, const int* idx, int count,
                             uint64_t* states, DevEvent* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= count) return;
  const int slot = slots[k], t = idx[slot];
  DevEvent e{};
  e.kind = 0;
  e.conductor = -1;
  e.dispatch = 3;
  e.point[0] = W.p[3 * slot];
  e.point[1] = W.p[3 * slot + 1];
  e.point[2] = W.p[3 * slot + 2];
  out[t] = e;
  states[t] = W.rng[slot];
}

size_t fdm_smem_bytes(int n, int Pn, bool psm) {
  const size_t m = static_cast<size_t>(n) * n * n;
  return 8 * static_cast<size_t>(Pn) * (1 + 2 * Pn) + (psm ? 8 * m : 0) + m;
}

// ---- geometry queries (the Structure API on the device, for unit parity) ---
// Per point: Structure::conductor_at(p, tol) (geometry.cpp:57-62, declaration
// index or -1), max_free_cube (:64-80; -1 where the reference throws),
// permittivity_at (:47-55; NaN outside the world) and the walk engine's
// fused transition prologue hop_scan (engine.cpp:293-298: conductor index,
// -1 grounded wall, -2 error, -3 free cube of half width hop_h).
__global__ void k_geometry(DStruct s, const double* pts, int count, double tol, int32_t* cond,
                           double* free_h, double* eps, int32_t* hop, double* hop_h) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  const double p[3] = {pts[3 * t], pts[3 * t + 1], pts[3 * t + 2]};
  cond[t] = conductor_at(s, p, tol);
  double h = -1.0;
  free_h[t] = max_free_cube(s, p, &h) ? h : -1.0;
  const int c = eps_class_at(s, p);
  eps[t] = c < 0 ? __longlong_as_double(0x7FF8000000000000ll) : __ldg(s.pal + c);
  double hh = -1.0;
  hop[t] = hop_scan(s, p, tol, &hh);
  hop_h[t] = hh;
}

// Per cube: the stratification probe + profile key of a transition cube
// (stratified_profile, geometry.cpp:357-396, then profile_key,
// sgf_cache.cpp:29-51): key axis (-1 general cube) and rounded layers.
__global__ void k_strat_keys(DStruct s, const double* cubes, int count, int n, int32_t* axis,
                             double* layers) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  const double c[3] = {cubes[4 * t], cubes[4 * t + 1], cubes[4 * t + 2]};
  const double h = cubes[4 * t + 3];
  const Prof P = strat_probe(s, c, h, n);
  axis[t] = P.axis;
  for (int q = 0; q < n; ++q)
    layers[static_cast<size_t>(t) * n + q] = P.axis >= 0 ? prof_layer(s, P, c, h, n, q) : 0.0;
}

// ---- deterministic tallies -------------------------------------------------
constexpr int kChunk = 1024;

// per block of kChunk walk records: per-slot sums in walk order
__global__ void __launch_bounds__(256)
    k_reduce_chunks(const WalkRec* recs, long long count, int nslots, double* psum,
                    double* psq, unsigned long long* pland, unsigned long long* pstat) {
  __shared__ int sl[kChunk];
  __shared__ double wt[kChunk];
  const long long base = static_cast<long long>(blockIdx.x) * kChunk;
  const int m = static_cast<int>(min(static_cast<long long>(kChunk), count - base));
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    sl[i] = recs[base + i].slot;
    wt[i] = recs[base + i].weight;
  }
  __syncthreads();
  for (int slot = threadIdx.x; slot < nslots; slot += blockDim.x) {
    double s1 = 0, s2 = 0;
    unsigned long long c = 0;
    for (int i = 0; i < m; ++i)
      if (sl[i] == slot) {
        const double w = wt[i];
        s1 += w;
        s2 += w * w;
        ++c;
      }
    psum[static_cast<size_t>(blockIdx.x) * nslots + slot] = s1;
    psq[static_cast<size_t>(blockIdx.x) * nslots + slot] = s2;
    pland[static_cast<size_t>(blockIdx.x) * nslots + slot] = c;
  }
  if (threadIdx.x == 0) {
    unsigned long long st[12] = {0};
    for (int i = 0; i < m; ++i) {
      const WalkRec& r = recs[base + i];
      st[0] += r.aborted;
      st[1] += r.resampled;
      if (r.branch < 4) st[2 + r.branch] += 1;
      st[6] += r.cached;
      st[7] += r.mw;
      st[8] += r.mw_steps;
    }
    for (int q = 0; q < 12; ++q) pstat[static_cast<size_t>(blockIdx.x) * 12 + q] = st[q];
  }
}

// pack: the call's tally as one f64 vector -- sum[nslots], sumsq[nslots],
// landed[nslots], stats[12] (counts exact below 2^53) -- the buffer
// frw_tally_allreduce combines across ranks with one NCCL all-reduce
__global__ void k_reduce_final(int nblocks, int nslots, const double* psum, const double* psq,
                               const unsigned long long* pland,
                               const unsigned long long* pstat, double* osum, double* osq,
                               unsigned long long* oland, unsigned long long* ostat,
                               double* pack) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nslots) {
    double s1 = 0, s2 = 0;
    unsigned long long c = 0;
    for (int b = 0; b < nblocks; ++b) {
      s1 += psum[static_cast<size_t>(b) * nslots + t];
      s2 += psq[static_cast<size_t>(b) * nslots + t];
      c += pland[static_cast<size_t>(b) * nslots + t];
    }
    osum[t] = s1;
    osq[t] = s2;
    oland[t] = c;
    pack[t] = s1;
    pack[nslots + t] = s2;
    pack[2 * nslots + t] = static_cast<double>(c);
  } else if (t < nslots + 12) {
    const int q = t - nslots;
    unsigned long long c = 0;
    for (int b = 0; b < nblocks; ++b) c += pstat[static_cast<size_t>(b) * 12 + q];
    ostat[q] = c;
    pack[3 * nslots + q] = static_cast<double>(c);
  }
}

// ---------------------------------------------------------------------------
// host side

double host_round_sig(double x, int digits) {  // sgf_cache.cpp:13-18
  if (x == 0 || !std::isfinite(x)) return x;
  const double e10 = std::floor(std::log10(std::fabs(x)));
  const double mag = std::pow(10.0, digits - 1 - e10);
  return std::round(x * mag) / mag;
}

template <class T>
T* dalloc(size_t n) {
  T* p = nullptr;
  if (cudaMalloc(&p, sizeof(T) * (n ? n : 1)) != cudaSuccess) return nullptr;
  return p;
}

struct SgfHost {
  int n = 0;
  int cap = 0;
  std::vector<uint64_t> hash;
  std::vector<int> entry;
  std::vector<int> axis;
  std::vector<double> keys;
  std::vector<double> pitch;
  std::vector<double*> data;  // device blocks
  // device mirrors
  uint64_t* d_hash = nullptr;
  int* d_entry = nullptr;
  int* d_axis = nullptr;
  double* d_keys = nullptr;
  double* d_pitch = nullptr;
  double** d_data = nullptr;
  size_t dev_entries_cap = 0;
  bool dirty = false;
  // uniform keys (axis 0, all layers equal): layer value -> first entry,
  // mirrored per palette class into d_uentry by uentry_sync
  std::map<double, int> uniform;
  int* d_uentry = nullptr;
  size_t uentry_cap = 0;
};

struct Engine {
  // structure
  int nc = 0, nd = 0, P = 0, bg = 0;
  double world[6];
  double *d_cbox = nullptr, *d_dbox = nullptr, *d_pal = nullptr, *d_alpha = nullptr,
         *d_rpal = nullptr;
  uint16_t* d_dcls = nullptr;
  bool have_structure = false;
  DGrid grid{};             // conductor bins (dims 0: none)
  int* d_cstart = nullptr;
  int* d_citem = nullptr;
  int* d_nstart = nullptr;
  int* d_nitem = nullptr;
  int* d_dstart = nullptr;
  int* d_ditem = nullptr;
  int* d_dlarge = nullptr;
  SgfHost sgf;
  // slots
  int S = 0;
  DSlots W{};
  WalkRec* recs = nullptr;
  long long recs_cap = 0;
  DCounters* d_cnt = nullptr;
  DMiss M{};
  int* mq[2] = {nullptr, nullptr};  // MicroWalk queues (current / next round)
  int* cq = nullptr;                // walks waiting for k_compile (this round)
  int* aq[2] = {nullptr, nullptr};  // ACTIVE queues (current / next round)
  int* ring_a = nullptr;  // k_flow rings of walk slots (-1 = empty entry)
  int* ring_m = nullptr;
  unsigned ring_mask = 0;
  cudaStream_t flow_stream = nullptr;  // the MicroWalk kernel of a two-kernel flow
  cudaEvent_t flow_fork = nullptr, flow_join = nullptr;
  // reduction scratch; `pack` holds the last call's tally (tally_n doubles)
  // for frw_tally_allreduce
  double* pack = nullptr;
  int tally_n = 0, tally_slots = 0, tally_mode = 0;
  long long tally_chunks = 0;  // kChunk-walk partial tallies of the last call (k_reduce_chunks)
  double *psum = nullptr, *psq = nullptr, *osum = nullptr, *osq = nullptr;
  unsigned long long *pland = nullptr, *pstat = nullptr, *oland = nullptr, *ostat = nullptr;
  size_t red_cap = 0;
  int red_slots = 0;
  // dense-hop voxel grids (k_mw_dense): one n^3 u16 grid per CTA
  uint16_t* dense_scratch = nullptr;
  size_t dense_cap = 0;
  // FDM solve scratch (5 Krylov vectors per persistent CTA)
  double* fdm_slab = nullptr;
  size_t fdm_cap = 0;
  std::vector<double> h_rpal;  // palette rounded to 6 significant digits (host copy)
  // lattice-jump tables (DJump) for lattice size jump_n, radii 2..jump_mmax
  int jump_n = 0, jump_mmax = 0;
  JumpMeta* d_jmeta = nullptr;
  uint64_t* d_jthr = nullptr;    // alias acceptance thresholds
  uint16_t* d_jguide = nullptr;  // aliases
};

void free_slots(Engine& E) {
  cudaFree(E.W.state);
  cudaFree(E.W.wid);
  cudaFree(E.W.p);
  cudaFree(E.W.weight);
  cudaFree(E.W.rng);
  cudaFree(E.W.hops);
  cudaFree(E.W.cached);
  cudaFree(E.W.mw);
  cudaFree(E.W.mwsteps);
  cudaFree(E.W.branch);
  cudaFree(E.W.resampled);
  cudaFree(E.W.cube);
  cudaFree(E.W.nbox);
  cudaFree(E.W.boxes);
  cudaFree(E.W.mwkind);
  cudaFree(E.W.atlas);
  cudaFree(E.mq[0]);
  cudaFree(E.mq[1]);
  E.mq[0] = E.mq[1] = nullptr;
  cudaFree(E.cq);
  E.cq = nullptr;
  cudaFree(E.W.mwnode);
  cudaFree(E.W.mwhsteps);
  cudaFree(E.W.mwhj);
  cudaFree(E.aq[0]);
  cudaFree(E.aq[1]);
  E.aq[0] = E.aq[1] = nullptr;
  cudaFree(E.ring_a);
  cudaFree(E.ring_m);
  E.ring_a = E.ring_m = nullptr;
  E.ring_mask = 0;
  if (E.flow_stream) cudaStreamDestroy(E.flow_stream);
  if (E.flow_fork) cudaEventDestroy(E.flow_fork);
  if (E.flow_join) cudaEventDestroy(E.flow_join);
  E.flow_stream = nullptr;
  E.flow_fork = E.flow_join = nullptr;
  cudaFree(E.M.retry);
  cudaFree(E.M.pend);
  cudaFree(E.M.park);
  cudaFree(E.M.dense);
  E.M.dense = nullptr;
  E.W = DSlots{};
  E.S = 0;
}

void engine_free(frw_ctx* ctx) {
  Engine* E = static_cast<Engine*>(ctx->walk);
  if (!E) return;
  cudaFree(E->d_cbox);
  cudaFree(E->d_cstart);
  cudaFree(E->d_citem);
  cudaFree(E->d_nstart);
  cudaFree(E->d_nitem);
  cudaFree(E->d_dstart);
  cudaFree(E->d_ditem);
  cudaFree(E->d_dlarge);
  cudaFree(E->d_dbox);
  cudaFree(E->d_pal);
  cudaFree(E->d_alpha);
  cudaFree(E->d_rpal);
  cudaFree(E->d_dcls);
  for (double* p : E->sgf.data) cudaFree(p);
  cudaFree(E->sgf.d_hash);
  cudaFree(E->sgf.d_entry);
  cudaFree(E->sgf.d_axis);
  cudaFree(E->sgf.d_keys);
  cudaFree(E->sgf.d_pitch);
  cudaFree(E->sgf.d_data);
  cudaFree(E->sgf.d_uentry);
  free_slots(*E);
  cudaFree(E->recs);
  cudaFree(E->d_cnt);
  cudaFree(E->M.axis);
  cudaFree(E->M.layers);
  cudaFree(E->psum);
  cudaFree(E->psq);
  cudaFree(E->pland);
  cudaFree(E->pstat);
  cudaFree(E->osum);
  cudaFree(E->osq);
  cudaFree(E->oland);
  cudaFree(E->ostat);
  cudaFree(E->pack);
  cudaFree(E->fdm_slab);
  cudaFree(E->dense_scratch);
  cudaFree(E->d_jmeta);
  cudaFree(E->d_jthr);
  cudaFree(E->d_jguide);
  delete E;
  ctx->walk = nullptr;
}

Engine* engine_of(frw_ctx* ctx) {
  if (!ctx->walk) {
    ctx->walk = new Engine;
    ctx->walk_free = engine_free;
  }
  return static_cast<Engine*>(ctx->walk);
}

uint64_t host_key_hash(int n, int axis, const double* layers) {  // == sgf_find's hash
  uint64_t h = (static_cast<uint64_t>(n) << 8) ^ static_cast<uint64_t>(axis);
  for (int t = 0; t < n; ++t) {
    uint64_t b;
    std::memcpy(&b, &layers[t], 8);
    h = key_step(h, b);
  }
  return sm64_mix(h);
}

int sgf_sync(frw_ctx* ctx, SgfHost& T) {
  if (!T.dirty) return FRW_OK;
  const size_t ne = T.axis.size();
  if (ne > T.dev_entries_cap || !T.d_axis) {
    const size_t cap = std::max<size_t>(64, ne * 2);
    cudaFree(T.d_axis);
    cudaFree(T.d_keys);
    cudaFree(T.d_pitch);
    cudaFree(T.d_data);
    T.d_axis = dalloc<int>(cap);
    T.d_keys = dalloc<double>(cap * NMAX);
    T.d_pitch = dalloc<double>(cap);
    T.d_data = dalloc<double*>(cap);
    if (!T.d_axis || !T.d_keys || !T.d_pitch || !T.d_data)
      return frw_fail(ctx, FRW_ENOMEM, "sgf table: device allocation failed");
    T.dev_entries_cap = cap;
  }
  cudaFree(T.d_hash);
  cudaFree(T.d_entry);
  T.d_hash = dalloc<uint64_t>(T.cap);
  T.d_entry = dalloc<int>(T.cap);
  FRW_CUDA(ctx, cudaMemcpyAsync(T.d_hash, T.hash.data(), 8 * T.cap, cudaMemcpyHostToDevice,
                                ctx->stream));
  FRW_CUDA(ctx, cudaMemcpyAsync(T.d_entry, T.entry.data(), 4 * T.cap, cudaMemcpyHostToDevice,
                                ctx->stream));
  if (ne) {
    FRW_CUDA(ctx, cudaMemcpyAsync(T.d_axis, T.axis.data(), 4 * ne, cudaMemcpyHostToDevice,
                                ctx->stream));
    FRW_CUDA(ctx, cudaMemcpyAsync(T.d_keys, T.keys.data(), 8 * ne * NMAX, cudaMemcpyHostToDevice,
                                ctx->stream));
    FRW_CUDA(ctx, cudaMemcpyAsync(T.d_pitch, T.pitch.data(), 8 * ne, cudaMemcpyHostToDevice,
                                ctx->stream));
    FRW_CUDA(ctx, cudaMemcpyAsync(T.d_data, T.data.data(), sizeof(double*) * ne,
                                  cudaMemcpyHostToDevice, ctx->stream));
  }
  T.dirty = false;
  return FRW_OK;
}

// per palette class: the table entry of its uniform key, or -1
int uentry_sync(frw_ctx* ctx, Engine& E) {
  SgfHost& T = E.sgf;
  const size_t P = std::max<size_t>(E.h_rpal.size(), 1);
  if (!T.d_uentry || T.uentry_cap < P) {
    cudaFree(T.d_uentry);
    T.d_uentry = dalloc<int>(P);
    T.uentry_cap = T.d_uentry ? P : 0;
    if (!T.d_uentry) return frw_fail(ctx, FRW_ENOMEM, "sgf table: device allocation failed");
  }
  std::vector<int> u(P, -1);
  for (size_t c = 0; c < E.h_rpal.size(); ++c) {
    const auto it = T.uniform.find(E.h_rpal[c]);
    if (it != T.uniform.end()) u[c] = it->second;
  }
  FRW_CUDA(ctx, cudaMemcpyAsync(T.d_uentry, u.data(), 4 * P, cudaMemcpyHostToDevice,
                                ctx->stream));
  return FRW_OK;
}

void sgf_insert_index(SgfHost& T, uint64_t h, int e) {
  if ((T.axis.size() + 1) * 2 > static_cast<size_t>(T.cap)) {
    const int ncap = std::max(256, T.cap * 2);
    std::vector<uint64_t> nh(ncap, 0);
    std::vector<int> ne(ncap, -1);
    for (int i = 0; i < T.cap; ++i)
      if (T.entry[i] >= 0) {
        int j = static_cast<int>(T.hash[i] & (ncap - 1));
        while (ne[j] >= 0) j = (j + 1) & (ncap - 1);
        nh[j] = T.hash[i];
        ne[j] = T.entry[i];
      }
    T.hash.swap(nh);
    T.entry.swap(ne);
    T.cap = ncap;
  }
  int j = static_cast<int>(h & (T.cap - 1));
  while (T.entry[j] >= 0) j = (j + 1) & (T.cap - 1);
  T.hash[j] = h;
  T.entry[j] = e;
}

DStruct make_dstruct(const Engine& E) {
  DStruct s{E.nc, E.nd, E.P, E.bg, E.d_cbox, E.d_dbox, E.d_dcls, E.d_pal, E.d_alpha, E.d_rpal,
            {}, E.grid};
  std::memcpy(s.world, E.world, sizeof s.world);
  return s;
}

DParams params_of(const frw_walk_params* prm) {
  DParams P{};
  P.n = prm->grid_n;
  P.panels = 6 * P.n * P.n;
  P.mode = prm->mode;
  P.rng = prm->rng_mode;
  P.snap = prm->snap;
  P.expansion = prm->expansion;
  P.hop_cap = prm->hop_cap;
  P.seed = prm->seed;
  P.mixed_seed = sm64_mix(prm->seed);
  std::memcpy(P.gbox, prm->gauss_box, sizeof P.gbox);
  std::memcpy(P.fcdf, prm->face_cdf, sizeof P.fcdf);
  P.area = prm->area_m2;
  return P;
}

// The face law f[v * s + u] (u, v = 0..s-1, s = 2m - 1; the six faces are
// equal) and E[tau] of the radius-m jump (see ensure_jumps).
void jump_law(int m, std::vector<long double>& f, long double& tot, long double& et) {
  const int side = 2 * m - 1, L = side + 1;
  const size_t K = static_cast<size_t>(side) * side;
  const long double pi = 3.141592653589793238462643383279502884L;
  std::vector<long double> phi(K), cs(side), pc(side), ps(side);
  for (int k = 1; k <= side; ++k) {
    cs[k - 1] = std::cos(pi * k / L);
    long double sum = 0;
    for (int i = 1; i <= side; ++i) {
      phi[(k - 1) * side + (i - 1)] = std::sqrt(2.0L / L) * std::sin(pi * k * i / L);
      sum += phi[(k - 1) * side + (i - 1)];
    }
    pc[k - 1] = phi[(k - 1) * side + (m - 1)];  // centre index m
    ps[k - 1] = sum;
  }
  // Bs[k2][k3] = sum_k1 phi_k1(1) phi_k1(c) phi_k2(c) phi_k3(c) / (6 (1 - lambda))
  std::vector<long double> Bs(K, 0.0L);
  et = 0;
  for (int k1 = 0; k1 < side; ++k1)
    for (int k2 = 0; k2 < side; ++k2)
      for (int k3 = 0; k3 < side; ++k3) {
        const long double inv = 1.0L / (1.0L - (cs[k1] + cs[k2] + cs[k3]) / 3.0L);
        Bs[k2 * side + k3] += phi[k1 * side] * pc[k1] * pc[k2] * pc[k3] * inv / 6.0L;
        et += pc[k1] * ps[k1] * pc[k2] * ps[k2] * pc[k3] * ps[k3] * inv;
      }
  // f[v][u] = sum_{k2,k3} phi_k2(u) Bs[k2][k3] phi_k3(v): the face law
  std::vector<long double> tmp(K, 0.0L);
  f.assign(K, 0.0L);
  for (int k2 = 0; k2 < side; ++k2)
    for (int v = 0; v < side; ++v) {
      long double acc = 0;
      for (int k3 = 0; k3 < side; ++k3) acc += Bs[k2 * side + k3] * phi[k3 * side + v];
      tmp[k2 * side + v] = acc;
    }
  tot = 0;
  for (int v = 0; v < side; ++v)
    for (int u = 0; u < side; ++u) {
      long double acc = 0;
      for (int k2 = 0; k2 < side; ++k2) acc += phi[k2 * side + u] * tmp[k2 * side + v];
      f[v * side + u] = std::max(acc, 0.0L);
      tot += f[v * side + u];
    }
}

// Lattice-jump tables (DJump) for lattice size n: radii m = 2..mmax with
// mmax = min((n - 1) / 2, 31, FRW_MW_JUMP); FRW_MW_JUMP=0 turns jumps off.
// The law of radius m is the simple symmetric walk's first hit of the
// sphere, i.e. its Green's function on the s^3 interior (s = 2m - 1, the
// sphere at indices 0 and s + 1 absorbing) next to a face.  That Green's
// function is diagonal in the DST-I basis phi_k(i) = sqrt(2/L) sin(pi k i/L),
// L = s + 1, with eigenvalue 1 - (cos(pi k1/L) + cos(pi k2/L) + cos(pi k3/L))/3,
// so P(hit (0, j, k)) = G((1, j, k), c) / 6 and E[tau] = sum_x G(x, c) are
// exact finite sums (O(s^3) per radius after factoring the k1 sum).
// (Not the reference SGF of a 2m-1 cube: its lattice faces step out with
// alpha 1, microwalk.cpp:97-104, while the sphere here sits inside a cell.)
int ensure_jumps(frw_ctx* ctx, Engine& E, int n, DJump* out) {
  int cap = 31;
  if (const char* e = std::getenv("FRW_MW_JUMP")) cap = std::atoi(e);
  const int mmax = std::min((n - 1) / 2, std::min(cap, 31));
  *out = DJump{};
  if (mmax < 2) return FRW_OK;
  if (E.jump_n != n || E.jump_mmax != mmax) {
    std::vector<JumpMeta> meta(mmax + 1, JumpMeta{});
    std::vector<uint64_t> prob;
    std::vector<uint16_t> alias;
    const long double two64 = 18446744073709551616.0L;
    for (int m = 2; m <= mmax; ++m) {
      const int side = 2 * m - 1;
      const size_t K = static_cast<size_t>(side) * side;
      std::vector<long double> f;
      long double tot = 0, et = 0;
      jump_law(m, f, tot, et);
      if (std::fabs(static_cast<double>(6.0L * tot) - 1.0) > 1e-9)
        return frw_fail(ctx, FRW_ESOLVE, "run_walks: lattice-jump law failed its normalisation");
      JumpMeta& jm = meta[m];
      jm.off = static_cast<uint32_t>(prob.size());
      jm.K = static_cast<uint32_t>(K);
      jm.side = static_cast<uint32_t>(side);
      jm.magic = static_cast<uint32_t>((4294967296ull + side - 1) / side);
      jm.esteps = static_cast<uint64_t>(static_cast<double>(et) * 4294967296.0 + 0.5);
      // Walker/Vose alias table of the face law: column i is kept with
      // probability q_i (scaled so the mean is 1), else its alias
      std::vector<long double> q(K);
      std::vector<size_t> small, large;
      for (size_t k = 0; k < K; ++k) {
        q[k] = f[k] / tot * static_cast<long double>(K);
        (q[k] < 1.0L ? small : large).push_back(k);
      }
      std::vector<uint64_t> pr(K, UINT64_MAX);
      std::vector<uint16_t> al(K);
      for (size_t k = 0; k < K; ++k) al[k] = static_cast<uint16_t>(k);
      while (!small.empty() && !large.empty()) {
        const size_t a = small.back(), b = large.back();
        small.pop_back();
        large.pop_back();
        const long double t = q[a] * two64;
        pr[a] = t >= two64 ? UINT64_MAX : static_cast<uint64_t>(t);
        al[a] = static_cast<uint16_t>(b);
        q[b] = (q[b] + q[a]) - 1.0L;
        (q[b] < 1.0L ? small : large).push_back(b);
      }
      // leftovers (rounding) keep their own column
      prob.insert(prob.end(), pr.begin(), pr.end());
      alias.insert(alias.end(), al.begin(), al.end());
    }
    cudaFree(E.d_jmeta);
    cudaFree(E.d_jthr);
    cudaFree(E.d_jguide);
    E.jump_n = 0;
    E.d_jmeta = dalloc<JumpMeta>(meta.size());
    E.d_jthr = dalloc<uint64_t>(prob.size());
    E.d_jguide = dalloc<uint16_t>(alias.size());
    if (!E.d_jmeta || !E.d_jthr || !E.d_jguide)
      return frw_fail(ctx, FRW_ENOMEM, "run_walks: jump table allocation failed");
    FRW_CUDA(ctx, cudaMemcpy(E.d_jmeta, meta.data(), sizeof(JumpMeta) * meta.size(),
                             cudaMemcpyHostToDevice));
    FRW_CUDA(ctx, cudaMemcpy(E.d_jthr, prob.data(), 8 * prob.size(), cudaMemcpyHostToDevice));
    FRW_CUDA(ctx, cudaMemcpy(E.d_jguide, alias.data(), 2 * alias.size(), cudaMemcpyHostToDevice));
    E.jump_n = n;
    E.jump_mmax = mmax;
  }
  out->mmax = mmax;
  // a second jump per Philox block measured 3-4% slower (C3/C5 HYBRID-MW):
  // more divergence between jumping and stepping lanes
  out->twice = 0;
  if (const char* e = std::getenv("FRW_MW_JUMP_TWICE")) out->twice = std::atoi(e);
  out->hom = 1;  // homogeneous-ball jumps (mw_hom_radius); FRW_MW_HOMJUMP=0 turns them off
  if (const char* e = std::getenv("FRW_MW_HOMJUMP")) out->hom = std::atoi(e);
  out->meta = E.d_jmeta;
  out->prob = E.d_jthr;  // (alias tables)
  out->alias = E.d_jguide;
  return FRW_OK;
}

// launches k_fdm over `Q` with enough persistent CTAs; scratch grows on demand
int launch_fdm(frw_ctx* ctx, Engine& E, const DStruct& s, const DParams& P, DCounters* C,
               const FdmQueue& Q) {
  const size_t cap = static_cast<size_t>(ctx->max_smem_optin);
  const bool psm = fdm_smem_bytes(P.n, kFdmClasses, true) <= cap;
  const size_t smem = fdm_smem_bytes(P.n, kFdmClasses, psm);
  if (smem > cap)
    return frw_fail(ctx, FRW_EINVAL, "FDM: lattice too large for the shared-memory class field");
  // one CTA per SM keeps every CTA's five Krylov vectors (5 x 8 n^3 bytes)
  // L2-resident: 148 x 553 KB at n = 24 against 126 MB of L2
  const int grid = ctx->sm_count;
  const size_t need = static_cast<size_t>(grid) * 5 * P.n * P.n * P.n;
  if (E.fdm_cap < need) {
    cudaFree(E.fdm_slab);
    E.fdm_slab = dalloc<double>(need);
    E.fdm_cap = E.fdm_slab ? need : 0;
    if (!E.fdm_slab) return frw_fail(ctx, FRW_ENOMEM, "FDM: scratch allocation failed");
  }
  auto kern = psm ? k_fdm<true> : k_fdm<false>;
  FRW_CUDA(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
  kern<<<grid, kFdmThreads, smem, ctx->stream>>>(s, P, E.W, C, Q, E.fdm_slab);
  FRW_CUDA(ctx, cudaGetLastError());
  return FRW_OK;
}

// Solves the distinct keys of `nmiss` recorded table misses (device solver,
// or the caller's callback) and inserts them; *added = new entries.
int resolve_misses(frw_ctx* ctx, Engine& E, int n, unsigned long long nmiss, frw_miss_fn miss,
                   void* user, int* added) {
  const DMiss& M = E.M;
  const int nm = static_cast<int>(std::min<unsigned long long>(nmiss, kMissMax));
  std::vector<int> maxis(nm);
  std::vector<double> mlayers(static_cast<size_t>(nm) * NMAX);
  FRW_CUDA(ctx, cudaMemcpy(maxis.data(), M.axis, 4 * nm, cudaMemcpyDeviceToHost));
  FRW_CUDA(ctx, cudaMemcpy(mlayers.data(), M.layers, 8 * size_t(nm) * NMAX,
                           cudaMemcpyDeviceToHost));
  std::unordered_map<uint64_t, int> seen;
  std::vector<int> uaxis;
  std::vector<double> ulayers;
  for (int q = 0; q < nm; ++q) {
    const double* L = &mlayers[static_cast<size_t>(q) * NMAX];
    const uint64_t h = host_key_hash(n, maxis[q], L);
    auto it = seen.find(h);
    if (it != seen.end() && maxis[it->second] == maxis[q] &&
        std::memcmp(&mlayers[static_cast<size_t>(it->second) * NMAX], L, 8 * n) == 0)
      continue;
    seen[h] = q;
    uaxis.push_back(maxis[q]);
    ulayers.insert(ulayers.end(), L, L + n);
  }
  const int before = static_cast<int>(E.sgf.axis.size());
  if (miss) {
    if (miss(user, n, static_cast<int>(uaxis.size()), uaxis.data(), ulayers.data()) != 0)
      return frw_fail(ctx, FRW_ESOLVE, "run_walks: miss callback failed");
  } else {  // solve on the device and insert
    const int cnt = static_cast<int>(uaxis.size());
    const size_t pan = 6ull * n * n;
    std::vector<double> pr(pan * cnt), ke(3 * pan * cnt), cdf(pan);
    if (int rc = frw_sgf_solve(ctx, n, cnt, uaxis.data(), ulayers.data(), pr.data(), ke.data()))
      return rc;
    for (int q = 0; q < cnt; ++q) {
      double run = 0;
      for (size_t b = 0; b < pan; ++b) cdf[b] = run += pr[q * pan + b];
      if (int rc = frw_sgf_put(ctx, n, uaxis[q], &ulayers[static_cast<size_t>(q) * n], 1.0,
                               &pr[q * pan], cdf.data(), &ke[3 * q * pan]))
        return rc;
    }
  }
  if (static_cast<int>(E.sgf.axis.size()) == before)
    return frw_fail(ctx, FRW_EMISS, "run_walks: miss callback added no table entry");
  *added = static_cast<int>(E.sgf.axis.size()) - before;
  if (int rc = sgf_sync(ctx, E.sgf)) return rc;
  return uentry_sync(ctx, E);
}

// device bytes of one resident walk slot (slot arrays, job, queues, rings,
// restart lists; ensure_slots)
constexpr size_t kSlotBytes = 4 + 1 + 8 + 24 + 8 + 8 + 4 + 4 + 4 + 8 + 1 + 1 + 32 + 2 + 8 * KMAX + 1 +
                              8 * kAtlasWords + 8 + 8 + 8 + 8 + 16 + 16 + 16 + 8 + 4;

// Slot capacity only grows: calls of different sizes (the short last chunk
// of a stopping rule, the single-transition API) reuse the pool, and the
// active pool size of a call is set per call (frw_run_walks: W.S).
int ensure_slots(frw_ctx* ctx, Engine& E, int S) {
  if (E.S >= S) return FRW_OK;
  free_slots(E);
  DSlots& W = E.W;
  W.S = S;
  W.jtail = S;
  // job entries: one per slot, then one per resident k_tail lane
  const size_t J = static_cast<size_t>(S) + static_cast<size_t>(ctx->sm_count) * kTailBlocks * 256;
  W.J = static_cast<int>(J);
  E.M.cap = S;
  W.state = dalloc<uint8_t>(S);
  W.wid = dalloc<long long>(S);
  W.p = dalloc<double>(3 * size_t(S));
  W.weight = dalloc<double>(S);
  W.rng = dalloc<uint64_t>(S);
  W.hops = dalloc<int>(S);
  W.cached = dalloc<uint32_t>(S);
  W.mw = dalloc<uint32_t>(S);
  W.mwsteps = dalloc<uint64_t>(S);
  W.branch = dalloc<uint8_t>(S);
  W.resampled = dalloc<uint8_t>(S);
  W.cube = dalloc<double>(4 * J);
  W.nbox = dalloc<uint16_t>(J);
  W.boxes = dalloc<uint64_t>(J * KMAX);
  W.mwkind = dalloc<uint8_t>(J);
  W.atlas = dalloc<uint64_t>(J * kAtlasWords);
  E.mq[0] = dalloc<int>(S);
  E.mq[1] = dalloc<int>(S);
  E.cq = dalloc<int>(S);
  W.mwnode = dalloc<uint32_t>(S);
  W.mwhsteps = dalloc<int>(S);
  W.mwhj = dalloc<uint64_t>(S);
  E.aq[0] = dalloc<int>(S);
  E.aq[1] = dalloc<int>(S);
  {
    // k_flow rings: every walk sits in at most one ring, and every waiting
    // lane holds at most one reservation, so 2S + resident lanes suffices
    unsigned cap = 1;
    while (cap < 2u * static_cast<unsigned>(S) + (1u << 20)) cap <<= 1;
    E.ring_a = dalloc<int>(cap);
    E.ring_m = dalloc<int>(cap);
    E.ring_mask = cap - 1;
  }
  E.M.retry = dalloc<long long>(2 * size_t(S));  // parks accumulate up to S/2 + S
  E.M.pend = dalloc<long long>(2 * size_t(S));
  E.M.park = dalloc<int>(2 * size_t(S));
  E.M.dense = dalloc<int>(S);
  if (!W.state || !W.wid || !W.p || !W.weight || !W.rng || !W.hops || !W.cached || !W.mw ||
      !W.mwsteps || !W.branch || !W.resampled || !W.cube || !W.nbox || !W.boxes ||
      !W.atlas || !W.mwkind || !E.mq[0] || !E.mq[1] || !E.cq || !W.mwnode || !W.mwhsteps || !W.mwhj || !E.aq[0] ||
      !E.aq[1] || !E.ring_a || !E.M.dense ||
      !E.ring_m || !E.M.retry || !E.M.pend || !E.M.park) {
    free_slots(E);
    return frw_fail(ctx, FRW_ENOMEM, "walk slots: device allocation failed");
  }
  cudaMemset(W.state, 0, S);  // fresh slots are free (never a stale carried hop)
  E.S = S;
  return FRW_OK;
}

}  // namespace
}  // namespace frw

using namespace frw;

namespace frw {
namespace {
// Shared driver of frw_first_transitions / frw_transitions: uploads the
// inputs, runs `launch` over the pending entries, resolves table misses and
// re-runs the entries that missed (they drew nothing), then copies back.
template <class Out, class Launch, class Post>
int run_single(frw_ctx* ctx, const frw_walk_params* prm, int count, const double* pts,
               const int32_t* axsign, uint64_t* states, frw_miss_fn miss, void* user, Out* out,
               Launch launch, Post post) {
  Engine& E = *engine_of(ctx);
  if (!E.have_structure) return frw_fail(ctx, FRW_EINVAL, "transitions: no structure uploaded");
  if (!prm || prm->grid_n < 2 || prm->grid_n > NMAX)
    return frw_fail(ctx, FRW_EINVAL, "transitions: grid_n must lie in [2, 128]");
  if (prm->mode == FRW_MODE_FDM && prm->grid_n > kFdmMaxN)
    return frw_fail(ctx, FRW_EINVAL, "transitions: FDM mode supports grid_n <= 32");
  if (count < 0 || (count > 0 && (!pts || !states || !out)))
    return frw_fail(ctx, FRW_EINVAL, "transitions: bad arguments");
  if (E.sgf.n && E.sgf.n != prm->grid_n)
    return frw_fail(ctx, FRW_EINVAL, "transitions: SGF table holds another lattice size");
  if (count == 0) return FRW_OK;
  FRW_CUDA(ctx, cudaSetDevice(ctx->device));
  if (E.S < count)
    if (int rc = ensure_slots(ctx, E, count)) return rc;
  if (E.recs_cap < count) {
    cudaFree(E.recs);
    E.recs = dalloc<WalkRec>(count);
    if (!E.recs) return frw_fail(ctx, FRW_ENOMEM, "transitions: record allocation failed");
    E.recs_cap = count;
  }
  E.W.count = count;
  if (!E.d_cnt) {
    E.d_cnt = dalloc<DCounters>(1);
    E.M.axis = dalloc<int>(kMissMax);
    E.M.layers = dalloc<double>(size_t(kMissMax) * NMAX);
  }
  if (int rc = sgf_sync(ctx, E.sgf)) return rc;
  if (int rc = uentry_sync(ctx, E)) return rc;
  const DStruct s = make_dstruct(E);
  DParams P = params_of(prm);
  P.rng = FRW_RNG_SPLITMIX_PARITY;  // the caller's SplitMix64 streams
  P.count = count;
  double* d_pts = dalloc<double>(3 * size_t(count));
  int32_t* d_ax = axsign ? dalloc<int32_t>(2 * size_t(count)) : nullptr;
  uint64_t* d_st = dalloc<uint64_t>(count);
  int* d_idx = dalloc<int>(count);
  int* d_rc = dalloc<int>(count);
  Out* d_out = dalloc<Out>(count);
  auto release = [&] {
    cudaFree(d_pts);
    cudaFree(d_ax);
    cudaFree(d_st);
    cudaFree(d_idx);
    cudaFree(d_rc);
    cudaFree(d_out);
  };
  if (!d_pts || (axsign && !d_ax) || !d_st || !d_idx || !d_rc || !d_out) {
    release();
    return frw_fail(ctx, FRW_ENOMEM, "transitions: device allocation failed");
  }
  std::vector<int> pend(count), rc(count);
  for (int t = 0; t < count; ++t) pend[t] = t;
  int status = FRW_OK;
  cudaStream_t st = ctx->stream;
  cudaMemcpyAsync(d_pts, pts, 24 * size_t(count), cudaMemcpyHostToDevice, st);
  if (axsign) cudaMemcpyAsync(d_ax, axsign, 8 * size_t(count), cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d_st, states, 8 * size_t(count), cudaMemcpyHostToDevice, st);
  for (int pass = 0; !pend.empty() && status == FRW_OK; ++pass) {
    if (pass > 64) {
      status = frw_fail(ctx, FRW_EMISS, "transitions: table misses keep recurring");
      break;
    }
    const int np = static_cast<int>(pend.size());
    DSgf T{E.sgf.cap, E.sgf.d_hash, E.sgf.d_entry, E.sgf.d_axis, E.sgf.d_keys, E.sgf.d_pitch,
           E.sgf.d_data, E.sgf.d_uentry};
    cudaMemcpyAsync(d_idx, pend.data(), 4 * size_t(np), cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(E.d_cnt, 0, sizeof(DCounters), st);
    launch(s, T, P, E, d_pts, d_ax, d_st, d_idx, np, d_rc, d_out);
    DCounters c;
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpyAsync(rc.data(), d_rc, 4 * size_t(np), cudaMemcpyDeviceToHost, st) !=
            cudaSuccess ||
        cudaMemcpyAsync(&c, E.d_cnt, sizeof c, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      status = frw_fail(ctx, FRW_ECUDA, "transitions: kernel failed");
      break;
    }
    if (c.err) {
      status = c.err == static_cast<unsigned long long>(-FRW_ESTEPCAP)
                   ? frw_fail(ctx, FRW_ESTEPCAP, "microwalk transit exceeded the step cap")
                   : frw_fail(ctx, FRW_EINVAL,
                              "transitions: point outside the world or inside a conductor");
      break;
    }
    status = post(s, P, E, d_idx, np, rc, d_st, d_out);
    if (status) break;
    std::vector<int> next;
    for (int q = 0; q < np; ++q)
      if (rc[q] == 2) next.push_back(pend[q]);
    if (!next.empty()) {
      int added = 0;
      status = resolve_misses(ctx, E, P.n, c.nmiss, miss, user, &added);
    }
    pend.swap(next);
  }
  if (status == FRW_OK &&
      (cudaMemcpyAsync(out, d_out, sizeof(Out) * count, cudaMemcpyDeviceToHost, st) !=
           cudaSuccess ||
       cudaMemcpyAsync(states, d_st, 8 * size_t(count), cudaMemcpyDeviceToHost, st) !=
           cudaSuccess ||
       cudaStreamSynchronize(st) != cudaSuccess))
    status = frw_fail(ctx, FRW_ECUDA, "transitions: copy-back failed");
  release();
  return status;
}
}  // namespace
}  // namespace frw

extern "C" {

int frw_upload_structure(frw_ctx* ctx, const frw_structure* s) {
  if (!ctx || !s) return FRW_EINVAL;
  if (s->n_cond < 1 || s->n_diel < 0 || !s->cond_box || (s->n_diel > 0 && (!s->diel_box || !s->diel_eps)))
    return frw_fail(ctx, FRW_EINVAL, "upload_structure: malformed structure");
  FRW_CUDA(ctx, cudaSetDevice(ctx->device));
  Engine& E = *engine_of(ctx);
  // palette of distinct permittivities (background first)
  std::vector<double> pal{s->background_eps};
  std::vector<uint16_t> dcls(s->n_diel);
  std::unordered_map<uint64_t, int> index;  // palette by bit pattern
  {
    uint64_t bits;
    std::memcpy(&bits, &s->background_eps, 8);
    index.emplace(bits, 0);
  }
  for (int d = 0; d < s->n_diel; ++d) {
    const double e = s->diel_eps[d];
    uint64_t bits;
    std::memcpy(&bits, &e, 8);
    auto it = index.find(bits);
    int k;
    if (it != index.end()) {
      k = it->second;
    } else {
      if (pal.size() > static_cast<size_t>(kClassMax))
        return frw_fail(ctx, FRW_EINVAL, "upload_structure: more than 32767 distinct permittivities");
      k = static_cast<int>(pal.size());
      pal.push_back(e);
      index.emplace(bits, k);
    }
    dcls[d] = static_cast<uint16_t>(k);
  }
  const int P = static_cast<int>(pal.size());
  // the pair-alpha table for palettes that fit shared memory (larger ones
  // divide per cell change, lane_alphas)
  const int PA = P <= PMAX ? P : 1;
  std::vector<double> alpha(static_cast<size_t>(PA) * PA, 0.0), rpal(P);
  for (int a = 0; a < P; ++a) {
    rpal[a] = host_round_sig(pal[a], 6);
    if (P <= PMAX)
      for (int b = 0; b < P; ++b) alpha[a * P + b] = pal[a] / (pal[a] + pal[b]);
  }
  cudaFree(E.d_cbox);
  cudaFree(E.d_dbox);
  cudaFree(E.d_pal);
  cudaFree(E.d_alpha);
  cudaFree(E.d_rpal);
  cudaFree(E.d_dcls);
  E.d_cbox = dalloc<double>(6 * size_t(s->n_cond));
  E.d_dbox = dalloc<double>(6 * size_t(s->n_diel));
  E.d_dcls = dalloc<uint16_t>(s->n_diel);
  E.d_pal = dalloc<double>(P);
  E.d_alpha = dalloc<double>(size_t(PA) * PA);
  E.d_rpal = dalloc<double>(P);
  if (!E.d_cbox || !E.d_dbox || !E.d_dcls || !E.d_pal || !E.d_alpha || !E.d_rpal)
    return frw_fail(ctx, FRW_ENOMEM, "upload_structure: device allocation failed");
  FRW_CUDA(ctx, cudaMemcpyAsync(E.d_cbox, s->cond_box, 48 * size_t(s->n_cond), cudaMemcpyHostToDevice,
                                ctx->stream));
  if (s->n_diel) {
    FRW_CUDA(ctx, cudaMemcpyAsync(E.d_dbox, s->diel_box, 48 * size_t(s->n_diel), cudaMemcpyHostToDevice,
                                ctx->stream));
    FRW_CUDA(ctx, cudaMemcpyAsync(E.d_dcls, dcls.data(), 2 * size_t(s->n_diel),
                                  cudaMemcpyHostToDevice, ctx->stream));
  }
  FRW_CUDA(ctx, cudaMemcpyAsync(E.d_pal, pal.data(), 8 * P, cudaMemcpyHostToDevice,
                                ctx->stream));
  FRW_CUDA(ctx, cudaMemcpyAsync(E.d_alpha, alpha.data(), 8 * size_t(PA) * PA,
                                cudaMemcpyHostToDevice, ctx->stream));
  E.h_rpal = rpal;
  FRW_CUDA(ctx, cudaMemcpyAsync(E.d_rpal, rpal.data(), 8 * P, cudaMemcpyHostToDevice,
                                ctx->stream));
  // conductor bins for many-conductor structures (C5: 200 conductors)
  cudaFree(E.d_cstart);
  cudaFree(E.d_citem);
  cudaFree(E.d_nstart);
  cudaFree(E.d_nitem);
  cudaFree(E.d_dstart);
  cudaFree(E.d_ditem);
  cudaFree(E.d_dlarge);
  E.d_cstart = E.d_citem = E.d_nstart = E.d_nitem = nullptr;
  E.d_dstart = E.d_ditem = E.d_dlarge = nullptr;
  E.grid = DGrid{};
  int grid_min = kGridMinConductors;  // FRW_GRID_MIN overrides (tests force the bins)
  if (const char* e = std::getenv("FRW_GRID_MIN")) grid_min = std::atoi(e);
  if (s->n_cond > grid_min) {
    DGrid g{};
    double ext[3], vol = 1;
    for (int a = 0; a < 3; ++a) {
      g.lo[a] = s->world[a];
      ext[a] = s->world[3 + a] - s->world[a];
      vol *= ext[a];
    }
    const double target = std::min(std::max(32.0 * s->n_cond, 512.0), 262144.0);
    const double b = std::cbrt(vol / target);
    g.bsmin = 1e300;
    for (int a = 0; a < 3; ++a) {
      g.dims[a] = static_cast<int>(std::min(256.0, std::max(1.0, std::round(ext[a] / b))));
      g.bs[a] = ext[a] / g.dims[a];
      g.ibs[a] = 1.0 / g.bs[a];
      g.bsmin = std::min(g.bsmin, g.bs[a]);
    }
    const size_t bins = static_cast<size_t>(g.dims[0]) * g.dims[1] * g.dims[2];
    auto bin1 = [&](int a, double x) {  // bin_of, host copy of the same arithmetic
      const int i = static_cast<int>(std::floor((x - g.lo[a]) * g.ibs[a]));
      return std::min(std::max(i, 0), g.dims[a] - 1);
    };
    std::vector<int> count(bins + 1, 0), start(bins + 1, 0), item;
    for (int pass = 0; pass < 2; ++pass) {
      if (pass == 1) {
        for (size_t q = 0; q < bins; ++q) start[q + 1] = start[q] + count[q];
        item.assign(start[bins], 0);
        std::fill(count.begin(), count.end(), 0);
      }
      for (int c = 0; c < s->n_cond; ++c) {
        const double* bx = s->cond_box + 6 * c;
        const int x0 = bin1(0, bx[0]), x1 = bin1(0, bx[3]), y0 = bin1(1, bx[1]),
                  y1 = bin1(1, bx[4]), z0 = bin1(2, bx[2]), z1 = bin1(2, bx[5]);
        for (int z = z0; z <= z1; ++z)
          for (int y = y0; y <= y1; ++y)
            for (int x = x0; x <= x1; ++x) {
              const size_t bin = (static_cast<size_t>(z) * g.dims[1] + y) * g.dims[0] + x;
              if (pass == 1) item[start[bin] + count[bin]] = c;
              ++count[bin];
            }
      }
    }
    // Nearest candidates of a bin B (slightly inflated against rounding in
    // the point-to-bin map): with bound = min(min_c maxdist(B, c), an upper
    // bound of the wall distance over B), every conductor with
    // mindist(B, c) <= bound.  For p in B the nearest conductor c* has
    // mindist(B, c*) <= d(p, c*) <= d(p, c') <= maxdist(B, c') for all c',
    // and conductors beyond the wall distance cannot lower min(wall, d).
    std::vector<int> nstart(bins + 1, 0), nitem;
    {
      double wext = 0;
      for (int a = 0; a < 3; ++a) wext = std::max(wext, s->world[3 + a] - s->world[a]);
      const double slack = 1e-9 * wext;
      std::vector<double> mind(s->n_cond);
      for (int z = 0; z < g.dims[2]; ++z)
        for (int y = 0; y < g.dims[1]; ++y)
          for (int x = 0; x < g.dims[0]; ++x) {
            const int bi[3] = {x, y, z};
            double blo[3], bhi[3];
            for (int a = 0; a < 3; ++a) {
              blo[a] = g.lo[a] + bi[a] * g.bs[a] - slack;
              bhi[a] = g.lo[a] + (bi[a] + 1) * g.bs[a] + slack;
            }
            double wall = 1e300;  // upper bound of the wall distance over B
            for (int a = 0; a < 3; ++a) {
              const double wl = s->world[a], wh = s->world[3 + a], mid = 0.5 * (wl + wh);
              const double t = (blo[a] <= mid && mid <= bhi[a])
                                   ? 0.5 * (wh - wl)
                                   : std::max(std::min(blo[a] - wl, wh - blo[a]),
                                              std::min(bhi[a] - wl, wh - bhi[a]));
              wall = std::min(wall, t);
            }
            double bound = wall;
            for (int c = 0; c < s->n_cond; ++c) {
              const double* bx = s->cond_box + 6 * c;
              double mn = 0, mx = 0;
              for (int a = 0; a < 3; ++a) {
                mn = std::max(mn, std::max(bx[a] - bhi[a], blo[a] - bx[3 + a]));
                mx = std::max(mx, std::max(bx[a] - blo[a], bhi[a] - bx[3 + a]));
              }
              mind[c] = mn;
              bound = std::min(bound, mx);
            }
            const size_t bin = (static_cast<size_t>(z) * g.dims[1] + y) * g.dims[0] + x;
            for (int c = 0; c < s->n_cond; ++c)
              if (mind[c] <= bound + slack) nitem.push_back(c);
            nstart[bin + 1] = static_cast<int>(nitem.size());
          }
    }
    // dielectrics: those spanning more than a quarter of the bins (layers)
    // are always candidates; the others are listed in the bins they overlap
    std::vector<int> dlarge, dcount(bins, 0), dstart(bins + 1, 0), ditem;
    {
      std::vector<std::array<int, 6>> rng(s->n_diel);
      for (int d = 0; d < s->n_diel; ++d) {
        const double* bx = s->diel_box + 6 * d;
        rng[d] = {bin1(0, bx[0]), bin1(1, bx[1]), bin1(2, bx[2]),
                  bin1(0, bx[3]), bin1(1, bx[4]), bin1(2, bx[5])};
        const size_t cnt = static_cast<size_t>(rng[d][3] - rng[d][0] + 1) *
                           (rng[d][4] - rng[d][1] + 1) * (rng[d][5] - rng[d][2] + 1);
        if (cnt * 4 > bins) {
          dlarge.push_back(d);
          rng[d][0] = -1;  // not binned
        }
      }
      for (int pass = 0; pass < 2; ++pass) {
        if (pass == 1) {
          for (size_t q = 0; q < bins; ++q) dstart[q + 1] = dstart[q] + dcount[q];
          ditem.assign(dstart[bins], 0);
          std::fill(dcount.begin(), dcount.end(), 0);
        }
        for (int d = 0; d < s->n_diel; ++d) {
          if (rng[d][0] < 0) continue;
          for (int z = rng[d][2]; z <= rng[d][5]; ++z)
            for (int y = rng[d][1]; y <= rng[d][4]; ++y)
              for (int x = rng[d][0]; x <= rng[d][3]; ++x) {
                const size_t bin = (static_cast<size_t>(z) * g.dims[1] + y) * g.dims[0] + x;
                if (pass == 1) ditem[dstart[bin] + dcount[bin]] = d;
                ++dcount[bin];
              }
        }
      }
    }
    E.d_cstart = dalloc<int>(bins + 1);
    E.d_citem = dalloc<int>(std::max<size_t>(item.size(), 1));
    E.d_nstart = dalloc<int>(bins + 1);
    E.d_nitem = dalloc<int>(std::max<size_t>(nitem.size(), 1));
    E.d_dstart = dalloc<int>(bins + 1);
    E.d_ditem = dalloc<int>(std::max<size_t>(ditem.size(), 1));
    E.d_dlarge = dalloc<int>(std::max<size_t>(dlarge.size(), 1));
    if (!E.d_cstart || !E.d_citem || !E.d_nstart || !E.d_nitem || !E.d_dstart || !E.d_ditem ||
        !E.d_dlarge)
      return frw_fail(ctx, FRW_ENOMEM, "upload_structure: bin allocation failed");
    FRW_CUDA(ctx, cudaMemcpyAsync(E.d_dstart, dstart.data(), 4 * (bins + 1),
                                  cudaMemcpyHostToDevice, ctx->stream));
    if (!ditem.empty())
      FRW_CUDA(ctx, cudaMemcpyAsync(E.d_ditem, ditem.data(), 4 * ditem.size(),
                                    cudaMemcpyHostToDevice, ctx->stream));
    if (!dlarge.empty())
      FRW_CUDA(ctx, cudaMemcpyAsync(E.d_dlarge, dlarge.data(), 4 * dlarge.size(),
                                    cudaMemcpyHostToDevice, ctx->stream));
    g.dstart = E.d_dstart;
    g.ditem = E.d_ditem;
    g.dlarge = E.d_dlarge;
    g.ndlarge = static_cast<int>(dlarge.size());
    FRW_CUDA(ctx, cudaMemcpyAsync(E.d_cstart, start.data(), 4 * (bins + 1), cudaMemcpyHostToDevice,
                                  ctx->stream));
    if (!item.empty())
      FRW_CUDA(ctx, cudaMemcpyAsync(E.d_citem, item.data(), 4 * item.size(),
                                    cudaMemcpyHostToDevice, ctx->stream));
    FRW_CUDA(ctx, cudaMemcpyAsync(E.d_nstart, nstart.data(), 4 * (bins + 1),
                                  cudaMemcpyHostToDevice, ctx->stream));
    if (!nitem.empty())
      FRW_CUDA(ctx, cudaMemcpyAsync(E.d_nitem, nitem.data(), 4 * nitem.size(),
                                    cudaMemcpyHostToDevice, ctx->stream));
    FRW_CUDA(ctx, cudaStreamSynchronize(ctx->stream));  // host vectors go out of scope
    g.cstart = E.d_cstart;
    g.citem = E.d_citem;
    g.nstart = E.d_nstart;
    g.nitem = E.d_nitem;
    E.grid = g;
  }
  E.nc = s->n_cond;
  E.nd = s->n_diel;
  E.P = P;
  E.bg = 0;
  std::memcpy(E.world, s->world, sizeof E.world);
  E.have_structure = true;
  return FRW_OK;
}

int frw_sgf_put(frw_ctx* ctx, int n, int axis, const double* layers, double pitch,
                const double* probs, const double* cdf, const double* kernels) {
  if (!ctx || !layers || !probs || !cdf) return FRW_EINVAL;
  if (n < 1 || n > NMAX || axis < 0 || axis > 2)
    return frw_fail(ctx, FRW_EINVAL, "sgf_put: need 1 <= n <= 128 and 0 <= axis <= 2");
  FRW_CUDA(ctx, cudaSetDevice(ctx->device));
  Engine& E = *engine_of(ctx);
  SgfHost& T = E.sgf;
  if (T.n && T.n != n) return frw_fail(ctx, FRW_EINVAL, "sgf_put: one lattice size per table");
  T.n = n;
  const uint64_t h = host_key_hash(n, axis, layers);
  for (int i = static_cast<int>(h & (T.cap ? T.cap - 1 : 0)); T.cap; i = (i + 1) & (T.cap - 1)) {
    const int e = T.entry[i];
    if (e < 0) break;
    if (T.hash[i] == h && T.axis[e] == axis &&
        std::memcmp(&T.keys[static_cast<size_t>(e) * NMAX], layers, 8 * n) == 0)
      return FRW_OK;  // first stored result wins (sgf_cache.cpp:133-153)
  }
  const size_t panels = 6ull * n * n;
  // data block: cdf, probs, kernels[3], guide table (kGuide int32)
  double* blk = dalloc<double>(5 * panels + kGuide / 2);
  if (!blk) return frw_fail(ctx, FRW_ENOMEM, "sgf_put: device allocation failed");
  {
    std::vector<int> guide(kGuide);
    const double total = cdf[panels - 1];
    size_t i = 0;
    for (int b = 0; b < kGuide; ++b) {
      const double gb = (static_cast<double>(b) / kGuide) * total;
      while (i < panels && cdf[i] <= gb) ++i;  // first cdf > fl((b/G)*total)
      guide[b] = static_cast<int>(i);
    }
    FRW_CUDA(ctx, cudaMemcpyAsync(blk + 5 * panels, guide.data(), 4 * kGuide, cudaMemcpyHostToDevice,
                                ctx->stream));
  }
  FRW_CUDA(ctx, cudaMemcpyAsync(blk, cdf, 8 * panels, cudaMemcpyHostToDevice,
                                ctx->stream));
  FRW_CUDA(ctx, cudaMemcpyAsync(blk + panels, probs, 8 * panels, cudaMemcpyHostToDevice,
                                ctx->stream));
  if (kernels)
    FRW_CUDA(ctx, cudaMemcpyAsync(blk + 2 * panels, kernels, 24 * panels, cudaMemcpyHostToDevice,
                                ctx->stream));
  else
    FRW_CUDA(ctx, cudaMemsetAsync(blk + 2 * panels, 0, 24 * panels, ctx->stream));
  const int e = static_cast<int>(T.axis.size());
  T.axis.push_back(axis);
  T.keys.resize(static_cast<size_t>(e + 1) * NMAX, 0.0);
  std::memcpy(&T.keys[static_cast<size_t>(e) * NMAX], layers, 8 * n);
  T.pitch.push_back(pitch);
  T.data.push_back(blk);
  sgf_insert_index(T, h, e);
  if (axis == 0) {
    bool same = true;
    for (int t = 1; t < n && same; ++t) same = layers[t] == layers[0];
    if (same) T.uniform.emplace(layers[0], e);  // the first stored entry wins
  }
  T.dirty = true;
  return FRW_OK;
}

int frw_sgf_count(const frw_ctx* ctx, int* entries) {
  if (!ctx || !entries) return FRW_EINVAL;
  const Engine* E = static_cast<const Engine*>(ctx->walk);
  *entries = E ? static_cast<int>(E->sgf.axis.size()) : 0;
  return FRW_OK;
}

int frw_sgf_clear(frw_ctx* ctx) {
  if (!ctx) return FRW_EINVAL;
  Engine& E = *engine_of(ctx);
  for (double* p : E.sgf.data) cudaFree(p);
  SgfHost fresh;
  fresh.d_hash = E.sgf.d_hash;
  fresh.d_entry = E.sgf.d_entry;
  fresh.d_axis = E.sgf.d_axis;
  fresh.d_keys = E.sgf.d_keys;
  fresh.d_pitch = E.sgf.d_pitch;
  fresh.d_data = E.sgf.d_data;
  fresh.d_uentry = E.sgf.d_uentry;
  fresh.uentry_cap = E.sgf.uentry_cap;
  fresh.dev_entries_cap = E.sgf.dev_entries_cap;
  fresh.dirty = true;
  E.sgf = fresh;
  return FRW_OK;
}

static_assert(sizeof(WalkRec) == sizeof(frw_walk_record), "record layout");

static int structure_transits(frw_ctx* ctx, int n, int count, const double* cubes,
                              int with_conductors, const uint64_t* states, int rng, uint64_t seed,
                        int jumps, int32_t step_cap, frw_exit* out) {
  if (!ctx) return FRW_EINVAL;
  Engine& E = *engine_of(ctx);
  if (!E.have_structure) return frw_fail(ctx, FRW_EINVAL, "transits: no structure uploaded");
  if (n < 1 || n > NMAX) return frw_fail(ctx, FRW_EINVAL, "transits: n must lie in [1, 128]");
  if (count < 0 || (count > 0 && (!cubes || (!states && rng != FRW_RNG_PHILOX) || !out)))
    return frw_fail(ctx, FRW_EINVAL, "transits: bad arguments");
  if (count == 0) return FRW_OK;
  for (int t = 0; t < count; ++t)
    if (!(cubes[4 * t + 3] > 0))
      return frw_fail(ctx, FRW_EINVAL, "transits: cube half width must be > 0");
  FRW_CUDA(ctx, cudaSetDevice(ctx->device));
  if (E.S < count)
    if (int rc = ensure_slots(ctx, E, count)) return rc;
  if (!E.d_cnt) {
    E.d_cnt = dalloc<DCounters>(1);
    E.M.axis = dalloc<int>(kMissMax);
    E.M.layers = dalloc<double>(size_t(kMissMax) * NMAX);
  }
  double* d_cubes = dalloc<double>(4 * size_t(count));
  uint64_t* d_states = dalloc<uint64_t>(count);
  DevExit* d_out = dalloc<DevExit>(count);
  auto release = [&] {
    cudaFree(d_cubes);
    cudaFree(d_states);
    cudaFree(d_out);
  };
  if (!d_cubes || !d_states || !d_out) {
    release();
    return frw_fail(ctx, FRW_ENOMEM, "transits: device allocation failed");
  }
  const DStruct s = make_dstruct(E);
  DParams P{};
  P.n = n;
  P.panels = 6 * n * n;
  P.rng = rng;
  P.seed = seed;
  if (rng == FRW_RNG_PHILOX && jumps) {
    if (int rc = ensure_jumps(ctx, E, n, &P.jump)) {
      release();
      return rc;
    }
  }
  const int cap = step_cap > 0 ? step_cap : 1000 * n * n;  // microwalk.cpp:81
  int status = FRW_OK;
  do {
    if (cudaMemcpyAsync(d_cubes, cubes, 32 * size_t(count), cudaMemcpyHostToDevice,
                        ctx->stream) != cudaSuccess ||
        (states && cudaMemcpyAsync(d_states, states, 8 * size_t(count), cudaMemcpyHostToDevice,
                                   ctx->stream) != cudaSuccess) ||
        cudaMemsetAsync(E.d_cnt, 0, sizeof(DCounters), ctx->stream) != cudaSuccess ||
        // job t arms from slot t: no stale S_MW_CARRY state may resume it
        cudaMemsetAsync(E.W.state, 0, static_cast<size_t>(count), ctx->stream) != cudaSuccess) {
      status = frw_fail(ctx, FRW_ECUDA, "transits: copy failed");
      break;
    }
    if (rng == FRW_RNG_PHILOX)
      k_transits<FRW_RNG_PHILOX><<<(count + 127) / 128, 128, 0, ctx->stream>>>(
          s, P, E.W, E.d_cnt, d_cubes, d_states, count, with_conductors, cap, d_out);
    else
      k_transits<FRW_RNG_SPLITMIX_PARITY><<<(count + 127) / 128, 128, 0, ctx->stream>>>(
          s, P, E.W, E.d_cnt, d_cubes, d_states, count, with_conductors, cap, d_out);
    DCounters c;
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpyAsync(out, d_out, sizeof(DevExit) * count, cudaMemcpyDeviceToHost,
                        ctx->stream) != cudaSuccess ||
        cudaMemcpyAsync(&c, E.d_cnt, sizeof c, cudaMemcpyDeviceToHost, ctx->stream) !=
            cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
      status = frw_fail(ctx, FRW_ECUDA, "transits: kernel failed");
      break;
    }
    if (c.err == static_cast<unsigned long long>(-FRW_ESTEPCAP))
      status = frw_fail(ctx, FRW_ESTEPCAP,
                        "microwalk transit exceeded the step cap; the lattice is malformed");
    else if (c.err)
      status = frw_fail(ctx, FRW_EINVAL, "transits: more than 64 boxes reach into one cube");
  } while (false);
  release();
  return status;
}

int frw_structure_transits(frw_ctx* ctx, int n, int count, const double* cubes,
                           int with_conductors, const uint64_t* states, int32_t step_cap,
                           frw_exit* out) {
  return structure_transits(ctx, n, count, cubes, with_conductors, states,
                            FRW_RNG_SPLITMIX_PARITY, 0, 0, step_cap, out);
}

int frw_structure_transits_philox(frw_ctx* ctx, int n, int count, const double* cubes,
                                  int with_conductors, uint64_t seed, int jumps,
                                  int32_t step_cap, frw_exit* out) {
  return structure_transits(ctx, n, count, cubes, with_conductors, nullptr, FRW_RNG_PHILOX,
                            seed, jumps, step_cap, out);
}

int frw_geometry_queries(frw_ctx* ctx, int count, const double* points, double tol,
                         int32_t* conductor_at, double* free_half_width, double* eps,
                         int32_t* hop_code, double* hop_half_width) {
  if (!ctx) return FRW_EINVAL;
  Engine& E = *engine_of(ctx);
  if (!E.have_structure) return frw_fail(ctx, FRW_EINVAL, "geometry: no structure uploaded");
  if (count < 0 || (count > 0 && (!points || !conductor_at || !free_half_width || !eps ||
                                  !hop_code || !hop_half_width)))
    return frw_fail(ctx, FRW_EINVAL, "geometry: bad arguments");
  if (count == 0) return FRW_OK;
  FRW_CUDA(ctx, cudaSetDevice(ctx->device));
  const size_t n = static_cast<size_t>(count);
  double* d_p = dalloc<double>(3 * n);
  int32_t* d_c = dalloc<int32_t>(n);
  double* d_f = dalloc<double>(n);
  double* d_e = dalloc<double>(n);
  int32_t* d_hc = dalloc<int32_t>(n);
  double* d_hh = dalloc<double>(n);
  int status = FRW_OK;
  if (!d_p || !d_c || !d_f || !d_e || !d_hc || !d_hh) {
    status = frw_fail(ctx, FRW_ENOMEM, "geometry: device allocation failed");
  } else {
    cudaStream_t st = ctx->stream;
    const DStruct s = make_dstruct(E);
    cudaMemcpyAsync(d_p, points, 24 * n, cudaMemcpyHostToDevice, st);
    k_geometry<<<(count + 127) / 128, 128, 0, st>>>(s, d_p, count, tol, d_c, d_f, d_e, d_hc,
                                                      d_hh);
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpyAsync(conductor_at, d_c, 4 * n, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(free_half_width, d_f, 8 * n, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(eps, d_e, 8 * n, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(hop_code, d_hc, 4 * n, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(hop_half_width, d_hh, 8 * n, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      status = frw_fail(ctx, FRW_ECUDA, "geometry: kernel failed");
  }
  cudaFree(d_p);
  cudaFree(d_c);
  cudaFree(d_f);
  cudaFree(d_e);
  cudaFree(d_hc);
  cudaFree(d_hh);
  return status;
}

int frw_stratified_keys(frw_ctx* ctx, int n, int count, const double* cubes, int32_t* axis,
                        double* layers) {
  if (!ctx) return FRW_EINVAL;
  Engine& E = *engine_of(ctx);
  if (!E.have_structure) return frw_fail(ctx, FRW_EINVAL, "strat keys: no structure uploaded");
  if (n < 1 || n > NMAX) return frw_fail(ctx, FRW_EINVAL, "strat keys: n must lie in [1, 128]");
  if (count < 0 || (count > 0 && (!cubes || !axis || !layers)))
    return frw_fail(ctx, FRW_EINVAL, "strat keys: bad arguments");
  if (count == 0) return FRW_OK;
  FRW_CUDA(ctx, cudaSetDevice(ctx->device));
  const size_t m = static_cast<size_t>(count);
  double* d_c = dalloc<double>(4 * m);
  int32_t* d_a = dalloc<int32_t>(m);
  double* d_l = dalloc<double>(m * n);
  int status = FRW_OK;
  if (!d_c || !d_a || !d_l) {
    status = frw_fail(ctx, FRW_ENOMEM, "strat keys: device allocation failed");
  } else {
    cudaStream_t st = ctx->stream;
    const DStruct s = make_dstruct(E);
    cudaMemcpyAsync(d_c, cubes, 32 * m, cudaMemcpyHostToDevice, st);
    k_strat_keys<<<(count + 127) / 128, 128, 0, st>>>(s, d_c, count, n, d_a, d_l);
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpyAsync(axis, d_a, 4 * m, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(layers, d_l, 8 * m * n, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      status = frw_fail(ctx, FRW_ECUDA, "strat keys: kernel failed");
  }
  cudaFree(d_c);
  cudaFree(d_a);
  cudaFree(d_l);
  return status;
}

int frw_lattice_jump_law(int m, double* face, double* esteps) {
  if (m < 2 || m > 31 || !face) return FRW_EINVAL;
  std::vector<long double> f;
  long double tot = 0, et = 0;
  jump_law(m, f, tot, et);
  for (size_t k = 0; k < f.size(); ++k) face[k] = static_cast<double>(f[k]);
  if (esteps) *esteps = static_cast<double>(et);
  return FRW_OK;
}

int frw_first_transitions(frw_ctx* ctx, const frw_walk_params* prm, int count,
                          const double* gpoints, const int32_t* axis_sign, uint64_t* states,
                          frw_miss_fn miss, void* user, frw_first* out) {
  if (!ctx) return FRW_EINVAL;
  if (count > 0 && !axis_sign) return frw_fail(ctx, FRW_EINVAL, "first_transitions: axis_sign");
  return run_single(
      ctx, prm, count, gpoints, axis_sign, states, miss, user, reinterpret_cast<DevFirst*>(out),
      [&](const DStruct& s, const DSgf& T, const DParams& P, Engine& E, const double* pts,
          const int32_t* ax, uint64_t* st, const int* idx, int np, int* rc, DevFirst* o) {
        k_first_single<<<(np + 127) / 128, 128, 0, ctx->stream>>>(s, T, P, E.W, E.d_cnt, E.M, pts,
                                                                  ax, st, idx, np, rc, o);
      },
      [](const DStruct&, const DParams&, Engine&, const int*, int, const std::vector<int>&,
         uint64_t*, DevFirst*) { return FRW_OK; });
}

int frw_transitions(frw_ctx* ctx, const frw_walk_params* prm, int count, const double* points,
                    uint64_t* states, frw_miss_fn miss, void* user, frw_event* out) {
  if (!ctx) return FRW_EINVAL;
  return run_single(
      ctx, prm, count, points, nullptr, states, miss, user, reinterpret_cast<DevEvent*>(out),
      [&](const DStruct& s, const DSgf& T, const DParams& P, Engine& E, const double* pts,
          const int32_t*, uint64_t* st, const int* idx, int np, int* rc, DevEvent* o) {
        k_transition_single<<<(np + 127) / 128, 128, 0, ctx->stream>>>(
            s, T, P, E.W, E.recs, E.d_cnt, E.M, pts, st, idx, np, rc, o);
      },
      [&](const DStruct& s, const DParams& P, Engine& E, const int* d_idx, int np,
          const std::vector<int>& rc, uint64_t* d_st, DevEvent* d_out) -> int {
        // FDM jobs (rc 3): slot q holds the compiled cube of entry idx[q]
        std::vector<int> slots;
        for (int q = 0; q < np; ++q)
          if (rc[q] == 3) slots.push_back(q);
        if (slots.empty()) return FRW_OK;
        const int nf = static_cast<int>(slots.size());
        int* d_slots = dalloc<int>(nf);
        unsigned long long* d_q = dalloc<unsigned long long>(2);
        if (!d_slots || !d_q) {
          cudaFree(d_slots);
          cudaFree(d_q);
          return frw_fail(ctx, FRW_ENOMEM, "transitions: FDM queue allocation failed");
        }
        const unsigned long long qh[2] = {static_cast<unsigned long long>(nf), 0ull};
        cudaMemcpyAsync(d_slots, slots.data(), 4 * size_t(nf), cudaMemcpyHostToDevice, ctx->stream);
        cudaMemcpyAsync(d_q, qh, sizeof qh, cudaMemcpyHostToDevice, ctx->stream);
        const FdmQueue Q{d_slots, d_q, d_q + 1, nullptr, nullptr};
        int st = launch_fdm(ctx, E, s, P, E.d_cnt, Q);
        if (st == FRW_OK) {
          k_fdm_events<<<(nf + 127) / 128, 128, 0, ctx->stream>>>(E.W, d_slots, d_idx, nf, d_st,
                                                                  d_out);
          DCounters c;
          if (cudaMemcpyAsync(&c, E.d_cnt, sizeof c, cudaMemcpyDeviceToHost, ctx->stream) !=
                  cudaSuccess ||
              cudaStreamSynchronize(ctx->stream) != cudaSuccess)
            st = frw_fail(ctx, FRW_ECUDA, "transitions: FDM solve failed");
          else if (c.err)
            st = frw_fail(ctx, FRW_ESOLVE, "transition cube solve failed normalization check");
        }
        cudaFree(d_slots);
        cudaFree(d_q);
        return st;
      });
}

}  // extern "C"

// ---- NCCL (loaded at first use: the library does not link it, so a host
// process that already loaded its own libnccl.so.2 -- e.g. torch's -- shares
// that copy) ------------------------------------------------------------------
namespace frw {
namespace {
struct NcclApi {
  bool tried = false, ok = false;
  std::string why;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};
std::mutex g_nccl_mu;
NcclApi& nccl() {
  static NcclApi api;
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (api.tried) return api;
  api.tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    api.why = std::string("cannot load libnccl.so.2: ") + dlerror();
    return api;
  }
  api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
  api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
  api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
  api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
  api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
  api.ok = api.get_unique_id && api.comm_init_rank && api.all_reduce && api.comm_destroy &&
           api.error_string;
  if (!api.ok) api.why = "libnccl.so.2 lacks an expected symbol";
  return api;
}
int nccl_fail(frw_ctx* ctx, const char* what, ncclResult_t r) {
  return frw_fail(ctx, FRW_ECUDA, std::string(what) + ": " + nccl().error_string(r));
}
// the context's own communicator (frw_nccl_init); kept beside the walk engine
std::map<frw_ctx*, ncclComm_t>& comms() {
  static auto* m = new std::map<frw_ctx*, ncclComm_t>;
  return *m;
}
}  // namespace
}  // namespace frw

extern "C" {

int frw_nccl_unique_id(void* id) {
  if (!id) return FRW_EINVAL;
  NcclApi& api = nccl();
  if (!api.ok) return FRW_ECUDA;
  ncclUniqueId u;
  if (api.get_unique_id(&u) != ncclSuccess) return FRW_ECUDA;
  std::memcpy(id, &u, sizeof u);
  return FRW_OK;
}

int frw_nccl_init(frw_ctx* ctx, const void* id, int nranks, int rank) {
  if (!ctx || !id || nranks < 1 || rank < 0 || rank >= nranks) return FRW_EINVAL;
  NcclApi& api = nccl();
  if (!api.ok) return frw_fail(ctx, FRW_ECUDA, api.why);
  FRW_CUDA(ctx, cudaSetDevice(ctx->device));
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof u);
  ncclComm_t comm = nullptr;
  const ncclResult_t r = api.comm_init_rank(&comm, nranks, u, rank);
  if (r != ncclSuccess) return nccl_fail(ctx, "ncclCommInitRank", r);
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  auto& m = comms();
  if (m.count(ctx)) api.comm_destroy(m[ctx]);
  m[ctx] = comm;
  return FRW_OK;
}

int frw_nccl_destroy(frw_ctx* ctx) {
  if (!ctx) return FRW_EINVAL;
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  auto& m = comms();
  auto it = m.find(ctx);
  if (it == m.end()) return FRW_OK;
  nccl().comm_destroy(it->second);
  m.erase(it);
  return FRW_OK;
}

int frw_walk_chunk_tallies(frw_ctx* ctx, int64_t* nchunks, int32_t* chunk, double* sum,
                           double* sumsq, uint64_t* landed, uint64_t* stats) {
  if (!ctx || !nchunks) return FRW_EINVAL;
  Engine& E = *engine_of(ctx);
  if (E.tally_n == 0) return frw_fail(ctx, FRW_EINVAL, "chunk tallies: no successful run_walks");
  *nchunks = E.tally_chunks;
  if (chunk) *chunk = kChunk;
  const size_t ns = static_cast<size_t>(E.tally_chunks) * E.tally_slots;
  FRW_CUDA(ctx, cudaSetDevice(ctx->device));
  if (sum) FRW_CUDA(ctx, cudaMemcpyAsync(sum, E.psum, 8 * ns, cudaMemcpyDeviceToHost, ctx->stream));
  if (sumsq) FRW_CUDA(ctx, cudaMemcpyAsync(sumsq, E.psq, 8 * ns, cudaMemcpyDeviceToHost, ctx->stream));
  if (landed)
    FRW_CUDA(ctx, cudaMemcpyAsync(landed, E.pland, 8 * ns, cudaMemcpyDeviceToHost, ctx->stream));
  if (stats)
    FRW_CUDA(ctx, cudaMemcpyAsync(stats, E.pstat, 8 * 12 * static_cast<size_t>(E.tally_chunks),
                                  cudaMemcpyDeviceToHost, ctx->stream));
  FRW_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return FRW_OK;
}

int frw_tally_allreduce(frw_ctx* ctx, void* comm, frw_tally* out) {
  if (!ctx || !out) return FRW_EINVAL;
  Engine* E = static_cast<Engine*>(ctx->walk);
  if (!E || E->tally_n <= 0)
    return frw_fail(ctx, FRW_EINVAL, "tally_allreduce: no frw_run_walks tally on this context");
  NcclApi& api = nccl();
  if (!api.ok) return frw_fail(ctx, FRW_ECUDA, api.why);
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  if (!c) {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    auto it = comms().find(ctx);
    if (it != comms().end()) c = it->second;
  }
  if (!c) return frw_fail(ctx, FRW_EINVAL, "tally_allreduce: no communicator (frw_nccl_init)");
  FRW_CUDA(ctx, cudaSetDevice(ctx->device));
  // one all-reduce (sum) of the packed tally over NVLink / NVSwitch
  const ncclResult_t r = api.all_reduce(E->pack, E->pack, static_cast<size_t>(E->tally_n),
                                        ncclFloat64, ncclSum, c, ctx->stream);
  if (r != ncclSuccess) return nccl_fail(ctx, "ncclAllReduce", r);
  std::vector<double> h(E->tally_n);
  FRW_CUDA(ctx, cudaMemcpyAsync(h.data(), E->pack, 8 * h.size(), cudaMemcpyDeviceToHost,
                                ctx->stream));
  FRW_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  const int k = E->tally_slots;
  for (int i = 0; i < k; ++i) {
    if (out->sum) out->sum[i] = h[i];
    if (out->sumsq) out->sumsq[i] = h[k + i];
    if (out->landed) out->landed[i] = static_cast<uint64_t>(h[2 * k + i]);
  }
  const double* st = &h[3 * k];
  out->aborted = static_cast<uint64_t>(st[0]);
  out->resampled = static_cast<uint64_t>(st[1]);
  for (int b = 0; b < 4; ++b) out->first[b] = static_cast<uint64_t>(st[2 + b]);
  const bool mwe = E->tally_mode == FRW_MODE_MWE || E->tally_mode == FRW_MODE_HYBRID_MWE;
  const bool fdm = E->tally_mode == FRW_MODE_FDM;
  out->sub[0] = static_cast<uint64_t>(st[6]);
  out->sub[1] = mwe || fdm ? 0 : static_cast<uint64_t>(st[7]);
  out->sub[2] = mwe ? static_cast<uint64_t>(st[7]) : 0;
  out->sub[3] = fdm ? static_cast<uint64_t>(st[7]) : 0;
  out->mw_steps = static_cast<uint64_t>(st[8]);
  out->mw_jumps = static_cast<uint64_t>(st[9]);
  out->mw_jump_steps = static_cast<uint64_t>(st[10]);
  return FRW_OK;
}

int frw_run_walks(frw_ctx* ctx, const frw_walk_params* prm, int32_t master, uint64_t walk_begin,
                  int64_t count, frw_miss_fn miss, void* user, frw_tally* out,
                  frw_walk_record* records) {
  if (!ctx || !prm || !out) return FRW_EINVAL;
  Engine& E = *engine_of(ctx);
  if (!E.have_structure) return frw_fail(ctx, FRW_EINVAL, "run_walks: no structure uploaded");
  if (prm->grid_n < 2 || prm->grid_n > NMAX)
    return frw_fail(ctx, FRW_EINVAL, "run_walks: grid_n must lie in [2, 128]");
  if (prm->mode == FRW_MODE_FDM && prm->grid_n > kFdmMaxN)
    return frw_fail(ctx, FRW_EINVAL, "run_walks: FDM mode supports grid_n <= 32");
  if (prm->mode < FRW_MODE_FDM || prm->mode > FRW_MODE_HYBRID_MWE)
    return frw_fail(ctx, FRW_EINVAL, "run_walks: unknown mode");
  if (!(prm->expansion >= 1.0)) return frw_fail(ctx, FRW_EINVAL, "run_walks: expansion < 1");
  if (master < 0 || master >= E.nc) return frw_fail(ctx, FRW_EINVAL, "run_walks: bad master");
  if (count < 0) return frw_fail(ctx, FRW_EINVAL, "run_walks: count < 0");
  if (E.sgf.n && E.sgf.n != prm->grid_n)
    return frw_fail(ctx, FRW_EINVAL, "run_walks: SGF table holds another lattice size");
  FRW_CUDA(ctx, cudaSetDevice(ctx->device));
  E.tally_n = 0;  // no tally for frw_tally_allreduce until this call succeeds
  const int nslots = E.nc + 1;
  // resident walk slots: 2^20, or for long calls up to 2^22 (about half the
  // walks in flight: rounds stay full longer; 8M-walk calls run 3.1e7 ->
  // 3.7e7 walks/s on C3/C5 from 2^20 to 2^22 slots, ~10 GB of slot state).
  // An automatic pool is bounded by the free device memory and halved down
  // to the default when an allocation fails (several contexts or ranks may
  // share the GPU); capacity only grows, so mixed call sizes reuse it.
  int S = prm->n_slots > 0 ? prm->n_slots : kSlotsDefault;
  const bool auto_slots = prm->n_slots <= 0;
  if (auto_slots) {
    while (S < (1 << 22) && static_cast<long long>(S) * 2 < count) S *= 2;
    if (const char* e = std::getenv("FRW_SLOTS")) S = std::max(1024, std::atoi(e));
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) {
      const size_t have = static_cast<size_t>(E.S) * kSlotBytes;  // reusable pool
      while (S > kSlotsDefault && static_cast<size_t>(S) * kSlotBytes > (fr + have) / 2) S /= 2;
    }
  }
  {
    int rc = ensure_slots(ctx, E, S);
    while (rc == FRW_ENOMEM && auto_slots && S > kSlotsDefault) {
      cudaGetLastError();  // clear the failed allocation
      S /= 2;
      rc = ensure_slots(ctx, E, S);
    }
    if (rc) return rc;
  }
  DSlots Wc = E.W;  // the pool of this call: S active slots of the capacity
  Wc.S = S;
  Wc.count = count;
  if (E.recs_cap < count) {
    cudaFree(E.recs);
    E.recs = dalloc<WalkRec>(count);
    if (!E.recs) return frw_fail(ctx, FRW_ENOMEM, "run_walks: record allocation failed");
    E.recs_cap = count;
  }
  if (!E.d_cnt) {
    E.d_cnt = dalloc<DCounters>(1);
    E.M.axis = dalloc<int>(kMissMax);
    E.M.layers = dalloc<double>(size_t(kMissMax) * NMAX);
  }
  if (int rc = sgf_sync(ctx, E.sgf)) return rc;
  if (int rc = uentry_sync(ctx, E)) return rc;

  // events: created after every early-return allocation/sync step above and
  // destroyed on every exit below
  struct Events {
    cudaEvent_t t0 = nullptr, t1 = nullptr, m0 = nullptr, m1 = nullptr, a0 = nullptr, c0 = nullptr;
    ~Events() {
      for (cudaEvent_t e : {t0, t1, m0, m1, a0, c0})
        if (e) cudaEventDestroy(e);
    }
  } ev;
  cudaEventCreate(&ev.t0);
  cudaEventCreate(&ev.t1);
  cudaEventCreate(&ev.m0);
  cudaEventCreate(&ev.m1);
  // FRW_TRACE_ROUNDS=1: per-round queue lengths and stage times on stderr
  const bool trace = std::getenv("FRW_TRACE_ROUNDS") != nullptr;
  cudaEventCreate(&ev.a0);
  cudaEventCreate(&ev.c0);
  cudaEvent_t t0 = ev.t0, t1 = ev.t1, m0 = ev.m0, m1 = ev.m1, a0 = ev.a0, c0 = ev.c0;
  cudaEventRecord(t0, ctx->stream);

  const DStruct s = make_dstruct(E);
  DParams P = params_of(prm);
  P.walk_begin = walk_begin;
  P.count = count;
  P.master = master;
  DMiss M = E.M;
  // lattice jumps in plain MicroWalk hops only: MicroWalk-E cubes (with
  // their conductor faces) leave few jumps and lose 1-4% to the test
  bool jumps = P.mode != FRW_MODE_MWE && P.mode != FRW_MODE_HYBRID_MWE;
  if (const char* e = std::getenv("FRW_MWE_JUMPS")) jumps = jumps || std::atoi(e) != 0;
  if (P.rng == FRW_RNG_PHILOX && jumps)
    if (int rc = ensure_jumps(ctx, E, P.n, &P.jump)) return rc;

  {  // dense-hop grids (k_mw_dense), one per persistent CTA
    const size_t need = static_cast<size_t>(ctx->sm_count) * P.n * P.n * P.n;
    if (E.dense_cap < need) {
      cudaFree(E.dense_scratch);
      E.dense_scratch = dalloc<uint16_t>(need);
      E.dense_cap = E.dense_scratch ? need : 0;
      if (!E.dense_scratch) return frw_fail(ctx, FRW_ENOMEM, "run_walks: dense scratch allocation failed");
    }
  }
  FRW_CUDA(ctx, cudaMemsetAsync(E.W.state, 0, S, ctx->stream));
  FRW_CUDA(ctx, cudaMemsetAsync(E.recs, 0, sizeof(WalkRec) * count, ctx->stream));
  FRW_CUDA(ctx, cudaMemsetAsync(E.d_cnt, 0, sizeof(DCounters), ctx->stream));
  const int grid = ctx->sm_count * 8;
  const int adv_grid = ctx->sm_count * 4;  // persistent: 4 x 256 threads per SM
  const int mw_grid = ctx->sm_count * 2;   // persistent: 2 x 512 threads per SM
  // run-to-completion threshold (active walks); FRW_TAIL_WALKS overrides
  // (148 * 1024 after the box-scan cells: C3/C5 +7-8% over 148 * 2048; 100K-200K
  // within 1%, tools/tail_sweep2.sh)
  // tail kernel: k_flow with its roles split by SM (C3 +16%, C5 +25%
  // over k_tail); FRW_TAIL_KERNEL=tail selects k_tail, =flowwarp k_flow with roles by warp
  const char* tk = std::getenv("FRW_TAIL_KERNEL");
  const bool use_flow = !tk || std::strncmp(tk, "flow", 4) == 0;
  const bool flow_by_sm = use_flow && !(tk && std::strcmp(tk, "flowwarp") == 0);
  // =flow2: the two roles as two kernels on two streams (k_flow_adv, k_flow_mw)
  const bool flow_split = flow_by_sm && tk && std::strcmp(tk, "flow2") == 0;
  // threshold: k_flow runs hops about as efficiently as the rounds, so it takes over once
  // the rounds' slices stop filling the device (148 * 3072; 300K-700K within 2%,
  // tools/ab_flow3.sh); k_tail 148 * 1024 (100K-200K within 1%, tools/tail_sweep2.sh)
  unsigned long long tail_threshold =
      static_cast<unsigned long long>(ctx->sm_count) * (use_flow ? 3072 : 1024);
  if (const char* e = std::getenv("FRW_TAIL_WALKS")) tail_threshold = std::strtoull(e, nullptr, 10);
  // k_flow's share of transition SMs: the share of the rounds' time spent in k_spawn,
  // k_advance and k_compile (what its transition role does), measured on this run's own
  // rounds, times kFlowAdvBias; FRW_FLOW_ADV_PCT overrides (percent of the SMs)
  double adv_ms_acc = 0, mwk_ms_acc = 0;
  constexpr unsigned long long kFlowMinWalks = 8192;
  unsigned long long next_live = 0;  // walks entering the next pass of the loop
  constexpr double kFlowAdvBias = 1.05;
  P.flow_adv = 0;
  P.flow_sms = 0;
  // time slices of the wavefront rounds: a MicroWalk hop
  // gets kMwSlice super-steps per k_mw visit and a walk kAdvSlice
  // transitions per k_advance visit, then continues next round, so a round
  // costs its throughput, not its longest hop; FRW_MW_SLICE /
  // FRW_ADV_SLICE override (0: unlimited).
  P.mw_slice = P.mode == FRW_MODE_FDM ? 0 : kMwSlice;
  P.adv_slice = kAdvSlice;
  if (const char* e = std::getenv("FRW_MW_SLICE")) P.mw_slice = std::atoi(e);
  if (const char* e = std::getenv("FRW_ADV_SLICE")) P.adv_slice = std::atoi(e);
  {  // the box slices are dynamic shared memory beyond the 48 KB default
    static std::once_flag once;
    std::call_once(once, [] {
      cudaFuncSetAttribute(k_mw<FRW_RNG_PHILOX>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBoxSmem512);
      cudaFuncSetAttribute(k_mw<FRW_RNG_SPLITMIX_PARITY>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBoxSmem512);
      cudaFuncSetAttribute(k_tail<FRW_RNG_PHILOX>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBoxSmem256);
      cudaFuncSetAttribute(k_tail<FRW_RNG_SPLITMIX_PARITY>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBoxSmem256);
      cudaFuncSetAttribute(k_flow<FRW_RNG_PHILOX>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBoxSmem256);
      cudaFuncSetAttribute(k_flow<FRW_RNG_SPLITMIX_PARITY>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBoxSmem256);
      cudaFuncSetAttribute(k_flow_mw<FRW_RNG_PHILOX>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBoxSmem512);
      cudaFuncSetAttribute(k_flow_mw<FRW_RNG_SPLITMIX_PARITY>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBoxSmem512);
    });
  }
  bool tail = false;
  double mw_ms = 0;
  unsigned long long tail_cyc_mw0 = 0, tail_cyc_all0 = 0;
  uint64_t misses_total = 0, restarts = 0, resumes = 0;
  int status = FRW_OK;
  for (int round = 0;; ++round) {
    DSgf T{E.sgf.cap, E.sgf.d_hash, E.sgf.d_entry, E.sgf.d_axis, E.sgf.d_keys, E.sgf.d_pitch,
           E.sgf.d_data, E.sgf.d_uentry};
    int* aq_in = E.aq[round & 1];
    int* aq_out = E.aq[(round + 1) & 1];
    int* mq_in = E.mq[round & 1];
    int* mq_next = E.mq[(round + 1) & 1];
    cudaEventRecord(a0, ctx->stream);
    k_spawn<<<grid, 256, 0, ctx->stream>>>(s, T, P, Wc, E.recs, E.d_cnt, M, aq_in);
    if (tail) {
      cudaEventRecord(m0, ctx->stream);
      const int tb = ctx->sm_count * kTailBlocks;  // persistent, one wave
      // a small batch (the parked walks of a miss cycle, a short call) is latency-bound:
      // k_tail's one lane per walk has no handoffs (2048 walks: 5.9 ms against 8.4 ms;
      // equal at 16K; the flow wins from there: 131K walks 10.2 against 13.0 ms,
      // tools/small_calls.py)
      if (use_flow && next_live > kFlowMinWalks) {
        if (flow_by_sm) {
          double f = adv_ms_acc + mwk_ms_acc > 0
                         ? kFlowAdvBias * adv_ms_acc / (adv_ms_acc + mwk_ms_acc)
                         : 0.4;
          if (const char* e = std::getenv("FRW_FLOW_ADV_PCT")) f = std::atof(e) / 100.0;
          f = std::min(0.75, std::max(0.15, f));
          P.flow_sms = std::max(1, ctx->sm_count / 2);  // SM pairs
          P.flow_adv = std::max(1, static_cast<int>(f * P.flow_sms + 0.5));
          if (trace)
            std::fprintf(stderr, "  k_flow: %d of %d SM pairs run transitions\n", P.flow_adv, P.flow_sms);
        }
        // rings start empty (a run that stopped on an error may leave entries)
        FRW_CUDA(ctx, cudaMemsetAsync(E.ring_a, 0xFF, 4ull * (E.ring_mask + 1), ctx->stream));
        FRW_CUDA(ctx, cudaMemsetAsync(E.ring_m, 0xFF, 4ull * (E.ring_mask + 1), ctx->stream));
        k_flow_init<<<1, 1, 0, ctx->stream>>>(E.d_cnt);
        if (flow_split) {
          if (!E.flow_stream) {
            FRW_CUDA(ctx, cudaStreamCreateWithFlags(&E.flow_stream, cudaStreamNonBlocking));
            FRW_CUDA(ctx, cudaEventCreateWithFlags(&E.flow_fork, cudaEventDisableTiming));
            FRW_CUDA(ctx, cudaEventCreateWithFlags(&E.flow_join, cudaEventDisableTiming));
          }
          FRW_CUDA(ctx, cudaEventRecord(E.flow_fork, ctx->stream));
          FRW_CUDA(ctx, cudaStreamWaitEvent(E.flow_stream, E.flow_fork, 0));
          // more CTAs than fit: those landing on SMs of the other role exit at once
          const int ga = ctx->sm_count * FRW_FLOWADV_MINB * 2, gm = ctx->sm_count * 2 * 2;
          k_flow_adv<<<ga, 256, 0, ctx->stream>>>(s, T, P, Wc, E.recs, E.d_cnt, M, aq_in,
                                                  E.ring_a, E.ring_m, E.ring_mask);
          if (P.rng == FRW_RNG_PHILOX)
            k_flow_mw<FRW_RNG_PHILOX><<<gm, 512, kBoxSmem512, E.flow_stream>>>(
                s, P, Wc, E.recs, E.d_cnt, mq_in, E.ring_a, E.ring_m, E.ring_mask);
          else
            k_flow_mw<FRW_RNG_SPLITMIX_PARITY><<<gm, 512, kBoxSmem512, E.flow_stream>>>(
                s, P, Wc, E.recs, E.d_cnt, mq_in, E.ring_a, E.ring_m, E.ring_mask);
          FRW_CUDA(ctx, cudaEventRecord(E.flow_join, E.flow_stream));
          FRW_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, E.flow_join, 0));
        } else if (P.rng == FRW_RNG_PHILOX)
          k_flow<FRW_RNG_PHILOX><<<tb, 256, kBoxSmem256, ctx->stream>>>(
              s, T, P, Wc, E.recs, E.d_cnt, M, aq_in, mq_in, E.ring_a, E.ring_m, E.ring_mask);
        else
          k_flow<FRW_RNG_SPLITMIX_PARITY><<<tb, 256, kBoxSmem256, ctx->stream>>>(
              s, T, P, Wc, E.recs, E.d_cnt, M, aq_in, mq_in, E.ring_a, E.ring_m, E.ring_mask);
      } else if (P.rng == FRW_RNG_PHILOX)
        k_tail<FRW_RNG_PHILOX><<<tb, 256, kBoxSmem256, ctx->stream>>>(s, T, P, Wc, E.recs, E.d_cnt, M,
                                                           aq_in, mq_in);
      else
        k_tail<FRW_RNG_SPLITMIX_PARITY><<<tb, 256, kBoxSmem256, ctx->stream>>>(s, T, P, Wc, E.recs,
                                                                    E.d_cnt, M, aq_in, mq_in);
    } else {
      k_advance<<<adv_grid, 256, 0, ctx->stream>>>(s, T, P, Wc, E.recs, E.d_cnt, M, aq_in,
                                                   E.cq, aq_out);
      // T_MW includes building the lazy field (engine.cpp:322-324 brackets
      // microwalk_transit_lazy)
      cudaEventRecord(m0, ctx->stream);
      k_compile<<<ctx->sm_count * 8, 256, 0, ctx->stream>>>(s, P, Wc, E.d_cnt, M, E.cq, mq_in);
      cudaEventRecord(c0, ctx->stream);
      if (P.mode == FRW_MODE_FDM) {
        const FdmQueue Q{mq_in, &E.d_cnt->qlen, &E.d_cnt->qhead, aq_out, &E.d_cnt->a2len};
        if (int rc = launch_fdm(ctx, E, s, P, E.d_cnt, Q)) {
          status = rc;
          break;
        }
      } else if (P.rng == FRW_RNG_PHILOX)
        k_mw<FRW_RNG_PHILOX><<<mw_grid, 512, kBoxSmem512, ctx->stream>>>(s, P, Wc, E.recs, E.d_cnt,
                                                               mq_in, aq_out, mq_next);
      else
        k_mw<FRW_RNG_SPLITMIX_PARITY><<<mw_grid, 512, kBoxSmem512, ctx->stream>>>(
            s, P, Wc, E.recs, E.d_cnt, mq_in, aq_out, mq_next);
    }
    // hops with more than KMAX boxes in their cube (exits 0 at once if none)
    if (P.mode != FRW_MODE_FDM) {
      if (P.rng == FRW_RNG_PHILOX)
        k_mw_dense<FRW_RNG_PHILOX><<<ctx->sm_count, 256, 0, ctx->stream>>>(
            s, P, Wc, E.recs, E.d_cnt, M.dense, aq_out, E.dense_scratch);
      else
        k_mw_dense<FRW_RNG_SPLITMIX_PARITY><<<ctx->sm_count, 256, 0, ctx->stream>>>(
            s, P, Wc, E.recs, E.d_cnt, M.dense, aq_out, E.dense_scratch);
    }
    cudaEventRecord(m1, ctx->stream);
    FRW_CUDA(ctx, cudaGetLastError());
    DCounters c;
    FRW_CUDA(ctx, cudaMemcpyAsync(&c, E.d_cnt, sizeof c, cudaMemcpyDeviceToHost, ctx->stream));
    FRW_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    {
      float ms = 0;
      cudaEventElapsedTime(&ms, m0, m1);
      // T_MW: k_mw (and the dense hops) are MicroWalk only; of a k_tail
      // launch only its warps' share of cycles in MicroWalk super-steps
      if (tail) {
        const double f = c.tail_all_cyc > tail_cyc_all0
                             ? static_cast<double>(c.tail_mw_cyc - tail_cyc_mw0) /
                                   static_cast<double>(c.tail_all_cyc - tail_cyc_all0)
                             : 0.0;
        tail_cyc_mw0 = c.tail_mw_cyc;
        tail_cyc_all0 = c.tail_all_cyc;
        mw_ms += f * ms;
      } else {
        mw_ms += ms;
      }
      if (!tail) {  // the rounds' time split, for k_flow's role shares
        float ams = 0, cms = 0;
        cudaEventElapsedTime(&ams, a0, m0);
        cudaEventElapsedTime(&cms, m0, c0);
        adv_ms_acc += ams + cms;
        mwk_ms_acc += ms - cms;
      }
      if (trace) {
        float ams = 0;
        cudaEventElapsedTime(&ams, a0, m0);
        std::fprintf(stderr,
                     "round %d: active %llu mw %llu next-active %llu carried %llu dense %llu "
                     "done %llu misses %llu spawn+advance %.3f ms %s %.3f ms\n",
                     round, c.alen, c.qlen, c.a2len, c.q2len, c.dqlen, c.done, c.nmiss, ams,
                     tail ? "tail" : "mw", ms);
        if (tail)  // busy warp-cycles (work in hand) by role, in ms of one warp at the SM clock
          std::fprintf(stderr, "  tail busy warp-ms: transitions %.1f MicroWalk %.1f\n",
                       (c.tail_all_cyc - c.tail_mw_cyc) / (ctx->sm_clock_khz * 1.0),
                       c.tail_mw_cyc / (ctx->sm_clock_khz * 1.0));
      }
    }
    if (c.chk_line) {
      status = frw_fail(ctx, FRW_ECUDA, "device check failed at walk.cu:" +
                                            std::to_string(c.chk_line));
      break;
    }
    if (c.err) {
      status = -static_cast<int>(c.err);
      frw_fail(ctx, status,
               status == FRW_ESTEPCAP
                   ? "microwalk transit exceeded the step cap; the lattice is malformed"
                   : "walk engine: geometry error (point outside the world or inside a "
                     "conductor, or FDM mode on a cube with more than 64 boxes)");
      break;
    }
    const bool all_spawned = c.next >= static_cast<unsigned long long>(count) &&
                             c.pend_head >= c.npend;
    const bool idle = all_spawned && c.a2len == 0 && c.q2len == 0;
    // Table misses are resolved lazily: parked walks wait while the others
    // run on, so the keys of a whole run are solved in a few batches instead
    // of one host round trip per discovering round.  Resolve when nothing
    // else is left, or when the miss / park records fill up.
    if (c.nmiss && (idle || c.nmiss >= kMissMax ||
                    c.nretry + c.npark > static_cast<unsigned long long>(S) / 2)) {
      int added = 0;
      status = resolve_misses(ctx, E, P.n, c.nmiss, miss, user, &added);
      if (status) break;
      misses_total += added;
      // walks whose first transition missed restart from scratch (pend <-
      // retry); walks parked mid-walk resume: their slots join the next
      // round's ACTIVE queue.  The round transition happens here too.
      FRW_CUDA(ctx, cudaMemcpyAsync(M.pend, M.retry, 8 * c.nretry, cudaMemcpyDeviceToDevice,
                                    ctx->stream));
      FRW_CUDA(ctx, cudaMemcpyAsync(aq_out + c.a2len, M.park, 4 * c.npark,
                                    cudaMemcpyDeviceToDevice, ctx->stream));
      DCounters upd = c;
      upd.npend = c.nretry;
      upd.pend_head = 0;
      upd.nretry = 0;
      upd.nmiss = 0;
      upd.npark = 0;
      upd.alen = c.a2len + c.npark;
      next_live = upd.alen + c.q2len;
      upd.ahead = 0;
      upd.a2len = 0;
      upd.qlen = c.q2len;  // the carried MicroWalk hops open the next round's queue
      upd.qhead = 0;
      upd.q2len = 0;
      upd.dqlen = 0;
      upd.dqhead = 0;
      upd.cqlen = 0;
      FRW_CUDA(ctx, cudaMemcpyAsync(E.d_cnt, &upd, sizeof upd, cudaMemcpyHostToDevice,
                                    ctx->stream));
      restarts += c.nretry;
      resumes += c.npark;
      if (trace)
        std::fprintf(stderr, "  resolved %d keys; restart %llu, resume %llu (total resumed %llu)\n",
                     added, c.nretry, c.npark, static_cast<unsigned long long>(resumes));
      continue;
    }
    if (idle) {
      if (c.done < static_cast<unsigned long long>(count))
        status = frw_fail(ctx, FRW_ECUDA, "run_walks: lost walks (internal error)");
      break;
    }
    // few walks left: run them to completion in one launch
    if (all_spawned && c.a2len + c.q2len <= tail_threshold && P.mode != FRW_MODE_FDM)
      tail = true;
    next_live = c.a2len + c.q2len;
    k_round<<<1, 1, 0, ctx->stream>>>(E.d_cnt);
  }
  if (status == FRW_OK) {
    // deterministic tallies
    const int nblocks = static_cast<int>((count + kChunk - 1) / kChunk);
    if (E.red_cap < static_cast<size_t>(std::max(nblocks, 1)) * nslots || E.red_slots != nslots) {
      cudaFree(E.psum);
      cudaFree(E.psq);
      cudaFree(E.pland);
      cudaFree(E.pstat);
      cudaFree(E.osum);
      cudaFree(E.osq);
      cudaFree(E.oland);
      cudaFree(E.ostat);
      cudaFree(E.pack);
      const size_t cap = static_cast<size_t>(std::max(nblocks, 1)) * nslots;
      E.psum = dalloc<double>(cap);
      E.psq = dalloc<double>(cap);
      E.pland = dalloc<unsigned long long>(cap);
      E.pstat = dalloc<unsigned long long>(static_cast<size_t>(std::max(nblocks, 1)) * 12);
      E.osum = dalloc<double>(nslots);
      E.osq = dalloc<double>(nslots);
      E.oland = dalloc<unsigned long long>(nslots);
      E.ostat = dalloc<unsigned long long>(12);
      E.pack = dalloc<double>(3 * static_cast<size_t>(nslots) + 12);
      if (!E.psum || !E.psq || !E.pland || !E.pstat || !E.osum || !E.osq || !E.oland ||
          !E.ostat || !E.pack) {
        E.red_cap = 0;
        return frw_fail(ctx, FRW_ENOMEM, "run_walks: tally allocation failed");
      }
      E.red_cap = cap;
      E.red_slots = nslots;
    }
    std::vector<unsigned long long> st(12, 0);
    if (count > 0) {
      k_reduce_chunks<<<nblocks, 256, 0, ctx->stream>>>(E.recs, count, nslots, E.psum, E.psq,
                                                         E.pland, E.pstat);
      k_reduce_final<<<(nslots + 12 + 127) / 128, 128, 0, ctx->stream>>>(
          nblocks, nslots, E.psum, E.psq, E.pland, E.pstat, E.osum, E.osq, E.oland, E.ostat,
          E.pack);
      FRW_CUDA(ctx, cudaGetLastError());
      if (out->sum)
        FRW_CUDA(ctx, cudaMemcpyAsync(out->sum, E.osum, 8 * nslots, cudaMemcpyDeviceToHost,
                                      ctx->stream));
      if (out->sumsq)
        FRW_CUDA(ctx, cudaMemcpyAsync(out->sumsq, E.osq, 8 * nslots, cudaMemcpyDeviceToHost,
                                      ctx->stream));
      if (out->landed)
        FRW_CUDA(ctx, cudaMemcpyAsync(out->landed, E.oland, 8 * nslots, cudaMemcpyDeviceToHost,
                                      ctx->stream));
      FRW_CUDA(ctx, cudaMemcpyAsync(st.data(), E.ostat, 8 * 12, cudaMemcpyDeviceToHost,
                                    ctx->stream));
    } else {
      FRW_CUDA(ctx, cudaMemsetAsync(E.pack, 0, 8 * (3 * static_cast<size_t>(nslots) + 12),
                                    ctx->stream));
      for (int k = 0; k < nslots; ++k) {
        if (out->sum) out->sum[k] = 0;
        if (out->sumsq) out->sumsq[k] = 0;
        if (out->landed) out->landed[k] = 0;
      }
    }
    if (records && count > 0)
      FRW_CUDA(ctx, cudaMemcpyAsync(records, E.recs, sizeof(WalkRec) * count,
                                    cudaMemcpyDeviceToHost, ctx->stream));
    cudaEventRecord(t1, ctx->stream);
    FRW_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    E.tally_n = 3 * nslots + 12;
    E.tally_slots = nslots;
    E.tally_mode = P.mode;
    E.tally_chunks = count > 0 ? (count + kChunk - 1) / kChunk : 0;
    out->aborted = st[0];
    out->resampled = st[1];
    for (int b = 0; b < 4; ++b) out->first[b] = st[2 + b];
    const bool mwe = P.mode == FRW_MODE_MWE || P.mode == FRW_MODE_HYBRID_MWE;
    const bool fdm = P.mode == FRW_MODE_FDM;
    out->sub[0] = st[6];
    out->sub[1] = mwe || fdm ? 0 : st[7];
    out->sub[2] = mwe ? st[7] : 0;  // lattice hops count as microwalk_e in MWE mode
    out->sub[3] = fdm ? st[7] : 0;  // general cubes solved by FDM
    out->mw_steps = st[8];
    out->cache_misses = misses_total;
    out->cache_hits = 0;
    out->restarts = restarts;
    out->mw_ms = mw_ms;
    DCounters cfin;
    FRW_CUDA(ctx, cudaMemcpy(&cfin, E.d_cnt, sizeof cfin, cudaMemcpyDeviceToHost));
    out->mw_general_steps = cfin.gen_steps;
    out->mw_cell_changes = cfin.cell_chg;
    out->mw_jumps = cfin.jumps;
    out->mw_jump_steps = cfin.jsteps;
    out->mw_dense_hops = cfin.dense_hops;
    // the jump counters join the packed tally (stats slots 9, 10)
    const double js[2] = {static_cast<double>(cfin.jumps), static_cast<double>(cfin.jsteps)};
    FRW_CUDA(ctx, cudaMemcpy(E.pack + 3 * nslots + 9, js, sizeof js, cudaMemcpyHostToDevice));
    float tot = 0;
    cudaEventElapsedTime(&tot, t0, t1);
    out->total_ms = tot;
#ifdef FRW_PHASE_CLOCKS
    {
      std::vector<unsigned long long> rows(256 * 32);
      cudaMemcpyFromSymbol(rows.data(), g_ph, 8 * rows.size());
      unsigned long long ph[32] = {};
      for (int r = 0; r < 256; ++r)
        for (int i = 0; i < 32; ++i) ph[i] += rows[32 * r + i];
      static const char* nm[16] = {"hop_scan", "strat_probe", "cached_lookup_sample", "compile_job",
                                   "cell_change", "superstep", "tail_exit_reload", "-",
                                   "first_transition", "tail_adv_part", "tail_mw_part",
                                   "ss_philox", "ss_jump", "ss_steps", "ss_hom_radius", "-"};
      std::fprintf(stderr, "phase clocks (walks %lld, total %.3f ms):\n", static_cast<long long>(count), tot);
      for (int i = 0; i < 15; ++i) {
        const unsigned long long cnt = i == 9 || i == 10 ? ph[25] : ph[16 + i];
        if (cnt)
          std::fprintf(stderr, "  %-22s events %12llu  cycles/event %10.1f  total Gcyc %8.3f\n", nm[i],
                       cnt, static_cast<double>(ph[i]) / cnt, ph[i] * 1e-9);
      }
      std::fill(rows.begin(), rows.end(), 0ull);
      cudaMemcpyToSymbol(g_ph, rows.data(), 8 * rows.size());
      unsigned long long hist[256];
      cudaMemcpyFromSymbol(hist, g_tail_hist, sizeof hist);
      std::fprintf(stderr, "  k_tail completions per 0.25 ms (first launch from its start):");
      for (int i = 0; i < 256; ++i)
        if (hist[i]) std::fprintf(stderr, " %d:%llu", i, hist[i]);
      std::fprintf(stderr, "\n");
      std::memset(hist, 0, sizeof hist);
      cudaMemcpyToSymbol(g_tail_hist, hist, sizeof hist);
      const unsigned long long z = 0;
      const int zi = 0;
      cudaMemcpyToSymbol(g_tail_t0, &z, sizeof z);
      cudaMemcpyToSymbol(g_in_tail, &zi, sizeof zi);
    }
#endif
  }
  return status;
}

}  // extern "C"
