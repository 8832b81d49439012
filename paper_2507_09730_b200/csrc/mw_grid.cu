// mw_grid.cu -- single-cube MicroWalk on sm_100a (configs C1/C2).
//
// Reference semantics: walk_lattice<GridField> (proj/src/microwalk.cpp:
// 77-156) driven by microwalk_transit (microwalk.cpp:188-197), one
// SplitMix64(seed, stream) per transit in parity mode.
//
// B200 design:
//  * The cube is compiled once into a stencil table: every node gets a
//    16-bit id of its distinct "step record" (the six alphas of Eq. 5 depend
//    only on the node's and its neighbours' permittivities, so the C2 cube
//    has ~3k distinct records for 69k nodes).  A record carries the five
//    direction thresholds in the integer domain of the 53-bit uniform:
//    x >= X_d  <=>  fl(x*2^-53*sum) >= acc_d, with acc_d the reference's
//    in-order partial sums (microwalk.cpp:105-121).  Integer comparisons
//    against X_d reproduce the reference's f64 scan bit for bit, with no
//    division and no FP64 on the step path.
//  * On chip a record is ONE 64-bit word: the top 11 bits of the five
//    thresholds in 12-bit SWAR lanes (guard bit per lane).  One 64-bit
//    multiply-add of x11 against all five lanes and a popcount of the guard
//    bits give the direction; only on an 11-bit tie (~0.25% of steps per
//    lane) are the exact 53-bit thresholds read from global memory (L1/L2).
//  * Node map (2 B/node) + packed records (8 B/record) are staged into shared
//    memory with cp.async.bulk (TMA bulk-copy engine, mbarrier completion):
//    183 KB for C2.  In the fast path (mw_grid_fast) the map holds each
//    node's record as its shared byte address and the walker's position is
//    the address of its map entry, so a step is LDS.U16 -> LDS.64 -> SHFL
//    (stride) with no address arithmetic: ~19 instructions per step, bound
//    by the shared-memory wavefronts of the two random gathers.
//  * Persistent CTAs, one walker per thread, refilled from a global transit
//    counter; lanes step in phase-aligned super-steps (8 steps per Philox
//    call) so Philox blocks and exit bookkeeping are warp-uniform: a lane
//    whose transit ends is re-armed with the next transit at the next
//    super-step boundary instead of idling.
//  * Histogram (RED.64 to global), exact u64 step moments and optional
//    per-transit records are fused into the exit path; the exit panel is one
//    lookup in a per-absorbing-node table.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <unordered_map>
#include <vector>

#include "frw_internal.h"
#include "frw_rng.cuh"

namespace frw {
namespace {

// stride lookup by warp shuffle (lane d holds stride d) instead of a shared
// load: it keeps the step's shared-memory wavefronts to the two gathers
#ifndef FRW_STRIDE_SHFL
#define FRW_STRIDE_SHFL 1
#endif
// Philox 8-step blocks per super-step of mw_grid_fast (exit bookkeeping and
// the step cap test run once per super-step)
#ifndef FRW_GRID_PB
#define FRW_GRID_PB 1
#endif
constexpr int kThreads = 1024;
constexpr int kDirAxis[6] = {0, 0, 1, 1, 2, 2};
constexpr int kDirSign[6] = {-1, +1, -1, +1, -1, +1};

// SWAR layout of a packed record
constexpr int kLane = 12;                          // 11-bit threshold + guard
constexpr uint64_t kOnes = 0x0000001001001001ull | (1ull << 48);  // 1 in each of 5 lanes
constexpr uint64_t kGuard = kOnes << 11;           // guard bit of each lane (11,23,35,47,59)
constexpr int kTop = 2047;                         // 11-bit lane maximum
// the exit record: every guard bit plus bit 63, counted by the fast path's
// popcount as direction 6 (stride 0); the other paths test the id first
constexpr uint32_t kGuardLo = static_cast<uint32_t>(kGuard);
constexpr uint32_t kGuardHi = static_cast<uint32_t>(kGuard >> 32) | 0x80000000u;
constexpr uint64_t kExitRec = kGuard | (1ull << 63);

// ---------------------------------------------------------------------------
// host: compile the grid into node map + step records

struct Key {
  uint64_t a, b;
  bool operator==(const Key& o) const { return a == o.a && b == o.b; }
};

// smallest x in [0, 2^53] with fl(x * sum) >= acc * 2^53 (2^53 if none);
// fl(x*sum) is monotone in x, so "x >= X" <=> "not (target < acc)".  The
// quotient lands within a few units of X; the two walks settle it exactly.
__host__ __device__ uint64_t threshold_of(double acc, double sum) {
  const double target = acc * 9007199254740992.0;  // ldexp(acc, 53): exact
  constexpr uint64_t kTop = 1ull << 53;
  const auto ok = [&](uint64_t x) { return static_cast<double>(x) * sum >= target; };
  const double g = target / sum;
  uint64_t x = !(g > 0) ? 0 : (g >= static_cast<double>(kTop) ? kTop : static_cast<uint64_t>(g));
  if (ok(x)) {
    while (x > 0 && ok(x - 1)) --x;
  } else {
    while (x < kTop && !ok(x)) ++x;
  }
  return x;
}

// e / (e + e) is exactly 1/2 unless e + e overflows
__host__ __device__ inline bool same_eps_halves(double e) { return e <= 0x1.0p1022; }

// open-addressing map from a 112-bit stencil key to its record index
struct KeyTable {
  std::vector<Key> key;
  std::vector<uint32_t> val;
  uint64_t mask;
  explicit KeyTable(size_t expect) {
    size_t cap = 1024;
    while (cap < 2 * expect) cap <<= 1;
    key.resize(cap);
    val.assign(cap, 0xFFFFFFFFu);
    mask = cap - 1;
  }
  // index of the key, inserting `next` when absent (returns {index, fresh})
  std::pair<uint32_t, bool> find_or_insert(const Key& k, uint32_t next) {
    uint64_t h = sm64_mix(k.a ^ sm64_mix(k.b)) & mask;
    while (val[h] != 0xFFFFFFFFu) {
      if (key[h] == k) return {val[h], false};
      h = (h + 1) & mask;
    }
    key[h] = k;
    val[h] = next;
    return {next, true};
  }
};

struct Compiled {
  std::vector<uint16_t> map;
  std::vector<uint64_t> rec;   // [R] packed
  std::vector<uint64_t> full;  // [R][5] exact thresholds X_d
  std::vector<int32_t> exit_info;  // [(n+2)^3] see exit_info_of
};

// What absorbing padded node p means to a walker that lands on it: a halo
// face node has exactly one lattice neighbour, so it names one surface panel
// (sgf.hpp:34-36, sgf.cpp:13-30); a conductor voxel names its conductor
// (-2 - id).  Edge/corner halo nodes and lattice nodes are never landed on
// from outside (-1).
void exit_info_of(int n, const int32_t* mask, std::vector<int32_t>& info) {
  const int np = n + 2;
  info.assign(static_cast<size_t>(np) * np * np, -1);
  for (int k = 0; k < np; ++k)
    for (int j = 0; j < np; ++j)
      for (int i = 0; i < np; ++i) {
        const int h[3] = {i, j, k};
        int out = 0, ax = -1;
        for (int a = 0; a < 3; ++a)
          if (h[a] == 0 || h[a] == n + 1) ++out, ax = a;
        const size_t pv = (static_cast<size_t>(k) * np + j) * np + i;
        if (out == 0) {
          if (mask) {
            const int m = mask[((k - 1) * n + (j - 1)) * n + (i - 1)];
            if (m >= 0) info[pv] = -2 - m;
          }
          continue;
        }
        if (out != 1) continue;
        const int dir = 2 * ax + (h[ax] == n + 1 ? 1 : 0);
        int c[3] = {i - 1, j - 1, k - 1};
        c[ax] = h[ax] == 0 ? 0 : n - 1;  // the interior node stepped from
        const int uu = ax == 0 ? c[1] : c[0];
        const int vv = ax == 2 ? c[1] : c[2];
        info[pv] = (dir * n + vv) * n + uu;
      }
}

int compile_grid(frw_ctx* ctx, int n, const double* eps, const int32_t* mask,
                 Compiled& out) {
  const int nodes = n * n * n;
  std::unordered_map<uint64_t, uint32_t> pal_of;
  std::vector<double> pal;
  std::vector<uint32_t> node_pal(nodes);
  uint64_t last_bits = 0;
  uint32_t last_idx = 0xFFFFFFFFu;
  for (int v = 0; v < nodes; ++v) {
    const double e = eps[v];
    if (!(e > 0) || !std::isfinite(e))
      return frw_fail(ctx, FRW_EINVAL, "grid permittivities must be finite and > 0");
    uint64_t bits;
    std::memcpy(&bits, &e, 8);
    if (bits == last_bits && last_idx != 0xFFFFFFFFu) {  // runs of equal permittivity
      node_pal[v] = last_idx;
      continue;
    }
    auto it = pal_of.find(bits);
    if (it == pal_of.end()) {
      if (pal.size() >= 0xFFF0)
        return frw_fail(ctx, FRW_EINVAL, "more than 65520 distinct permittivities");
      it = pal_of.emplace(bits, static_cast<uint32_t>(pal.size())).first;
      pal.push_back(e);
    }
    node_pal[v] = it->second;
    last_bits = bits;
    last_idx = it->second;
  }
  constexpr uint32_t kSurface = 0xFFFF, kCond = 0xFFFE;
  KeyTable rec_of(std::min<size_t>(nodes, 1u << 16));
  uint32_t nrec = 0;
  // Padded map: a one-node halo around the lattice.  Halo nodes and conductor
  // voxels are absorbing: they map to the exit record, appended after the
  // step records once their count is known.
  const int np = n + 2;
  std::vector<uint32_t> pmap(static_cast<size_t>(np) * np * np, 0xFFFFFFFFu);
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        const int v = (k * n + j) * n + i;
        const size_t pv = (static_cast<size_t>(k + 1) * np + (j + 1)) * np + (i + 1);
        const bool self_cond = mask && mask[v] >= 0;
        if (self_cond) continue;  // conductor voxel: exit record
        uint32_t code[6];
        for (int d = 0; d < 6; ++d) {
          int nb[3] = {i, j, k};
          nb[kDirAxis[d]] += kDirSign[d];
          if (nb[kDirAxis[d]] < 0 || nb[kDirAxis[d]] >= n) {
            code[d] = kSurface;
            continue;
          }
          const int nv = (nb[2] * n + nb[1]) * n + nb[0];
          code[d] = (mask && mask[nv] >= 0) ? kCond : node_pal[nv];
        }
        uint32_t self = node_pal[v];
        // A node whose non-absorbing neighbours all share its permittivity e
        // steps with alphas e / (e + e) = 1/2 whatever e is: one record for
        // all of them (palette id 0 stands for e), so the walkers inside
        // uniform regions gather one shared-memory address (a broadcast)
        // instead of one per permittivity.
        if (same_eps_halves(pal[self]) && same_eps_halves(pal[0])) {
          bool uniform = true;
          for (int d = 0; d < 6; ++d)
            uniform = uniform && (code[d] == self || code[d] == kSurface || code[d] == kCond);
          if (uniform) {
            for (int d = 0; d < 6; ++d)
              if (code[d] == self) code[d] = 0;
            self = 0;
          }
        }
        Key key{(uint64_t(self) << 48) | (uint64_t(code[0]) << 32) |
                    (uint64_t(code[1]) << 16) | code[2],
                (uint64_t(code[3]) << 32) | (uint64_t(code[4]) << 16) | code[5]};
        const auto [r, fresh] = rec_of.find_or_insert(key, nrec);
        if (fresh) {
          if (r >= 0xFFFF)
            return frw_fail(ctx, FRW_EINVAL, "more than 65535 distinct stencil records");
          ++nrec;
          // microwalk.cpp:91-109: alphas (1 on absorbing faces) and their
          // in-order partial sums
          double acc[6], sum = 0;
          uint64_t packed = 0;
          const double ev = pal[self];
          for (int d = 0; d < 6; ++d) {
            double a = 1.0;
            if (code[d] != kSurface && code[d] != kCond) {
              const double en = pal[code[d]];
              a = en / (en + ev);
            }
            sum += a;
            acc[d] = sum;
          }
          for (int d = 0; d < 5; ++d) {
            const uint64_t X = threshold_of(acc[d], sum);
            out.full.push_back(X);
            // X = 2^53 (never reached) clamps to 2047: every x with top bits
            // 2047 then ties and the exact fallback decides
            const uint64_t t11 = std::min<uint64_t>(X >> 42, kTop);
            // stored pre-negated: lane = 2047 - T_d, so x11*ones + record
            // carries into the lane's guard bit exactly when x11 > T_d
            packed |= (kTop - t11) << (kLane * d);
          }
          out.rec.push_back(packed);
        }
        pmap[pv] = r;
      }
  // the exit record: never stepped from (an absorbed walker stops)
  out.rec.push_back(kExitRec);
  for (int d = 0; d < 5; ++d) out.full.push_back(1ull << 53);
  exit_info_of(n, mask, out.exit_info);
  out.map.resize(pmap.size());
  for (size_t q = 0; q < pmap.size(); ++q)
    out.map[q] = static_cast<uint16_t>(pmap[q] == 0xFFFFFFFFu ? nrec : pmap[q]);
  return FRW_OK;
}

// ---------------------------------------------------------------------------
// device

struct DevGrid {
  const uint16_t* map;  // [(n+2)^3] padded lattice: halo and conductor voxels -> exit
  const uint64_t* rec;  // [R+1] packed SWAR records, R = the exit record
  const uint64_t* full;
  const int32_t* mask;
  const int32_t* exit_info;  // [(n+2)^3] absorbing node -> panel / -2 - conductor
  int n;
  int np, npp;          // padded extents n+2, (n+2)^2
  int start_idx;        // padded index of start_node
  uint32_t exit_rec;    // R
  uint32_t map_bytes;  // padded to 16
  uint32_t rec_bytes;  // padded to 16
  float inv_np, inv_npp;
};

struct DevParams {
  uint64_t seed;
  uint64_t mixed_seed;
  uint64_t stream_begin;
  long long count;
  int step_cap;
  const uint64_t* states;  // FRW_RNG_SPLITMIX_STATES
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// shared-window address materialized once into a register (keeps ptxas
// from re-deriving it from SR_CgaCtaId inside the step loop)
__device__ __forceinline__ uint32_t smem_base(const void* p) {
  uint32_t a;
  asm volatile("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }"
               : "=r"(a)
               : "l"(p));
  return a;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  uint32_t v;  // zero-extended into a 32-bit register (no 16-bit merges)
  asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint64_t lds_u64(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ int lds_s32(uint32_t a) {
  int v;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

// Stage [src, src+bytes) into shared memory with the bulk-copy engine.
__device__ void bulk_stage(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  const uint32_t b = smem_u32(bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
                 : "memory");
    constexpr uint32_t kChunk = 32768;
    for (uint32_t off = 0; off < bytes; off += kChunk) {
      const uint32_t sz = min(kChunk, bytes - off);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
          "[%0], [%1], %2, [%3];" ::"r"(smem_u32(static_cast<char*>(dst) + off)),
          "l"(static_cast<const char*>(src) + off), "r"(sz), "r"(b)
          : "memory");
    }
  }
  __syncthreads();
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(b)
        : "memory");
  }
}

// q = v / d for 0 <= v < 2^24 via a float reciprocal and one correction
__device__ __forceinline__ int fdiv(int v, int d, float inv) {
  int q = __float2int_rz(static_cast<float>(v) * inv);
  const int r = v - q * d;
  if (r < 0)
    --q;
  else if (r >= d)
    ++q;
  return q;
}

template <int RNG, bool SMEM>
__global__ void __launch_bounds__(kThreads, 1)
    mw_grid_kernel(DevGrid g, DevParams p, unsigned long long* ctr, int* err,
                   int32_t* out_panel, int32_t* out_steps, int32_t* out_cond,
                   long long* out_nd, unsigned long long* hist, unsigned long long* m_sum,
                   unsigned long long* m_sq, unsigned long long* m_cx) {
  // SplitMix64 draws (parity streams or caller states) vs Philox words
  constexpr bool SM = RNG != FRW_RNG_PHILOX;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ int stride[6];

  if (SMEM) bulk_stage(smem, g.map, g.map_bytes + g.rec_bytes, &bar);
  if (threadIdx.x < 6) {
    const int d = threadIdx.x, ax = d >> 1;
    stride[d] = ((d & 1) ? 1 : -1) * (ax == 0 ? 1 : ax == 1 ? g.np : g.npp);
  }
  __syncthreads();
  const uint32_t s_map = smem_base(smem);
  const uint32_t s_rec = s_map + g.map_bytes;
  const uint32_t s_str = smem_base(stride);

  const int n = g.n;
  const int cap = p.step_cap;
  const uint32_t kExit = g.exit_rec;
  unsigned long long ssum = 0, ssq = 0, cexit = 0;

  long long t = static_cast<long long>(atomicAdd(ctr, 1ull));
  long long t_next = static_cast<long long>(atomicAdd(ctr, 1ull));
  bool live = t < p.count;
  int idx = g.start_idx;
  int steps = 0;
  uint64_t sm = 0;   // parity: SplitMix64 state
  uint32_t blk = 0;  // philox: 8-step block index within the transit
  if (RNG == FRW_RNG_SPLITMIX_PARITY && live)
    sm = sm64_stream_from_mixed(p.mixed_seed, p.stream_begin + t);
  if (RNG == FRW_RNG_SPLITMIX_STATES && live) sm = p.states[t];
  const uint32_t k0 = static_cast<uint32_t>(p.seed);
  const uint32_t k1 = static_cast<uint32_t>(p.seed >> 32);

  // Philox: one 4x32-10 call per super-step of 8 steps -- each 32-bit word
  // gives two steps their top 16 bits of x; the low 37 bits are drawn from
  // the (id, step slot, 1) counter only when the 16-bit prefix ties a
  // threshold, so x is still an exact 53-bit uniform.  Parity: 4 steps.
  constexpr int SS = SM ? 4 : 8;
  int xdir = 0;  // direction of the last move
  while (__any_sync(0xFFFFFFFFu, live)) {
    // ---- one phase-aligned super-step of SS lattice steps ----------------
    uint32_t w[4];
    if (RNG == FRW_RNG_PHILOX) {
      const uint64_t id = static_cast<uint64_t>(p.stream_begin + t);
      const U32x4 o = philox4x32_10(
          {static_cast<uint32_t>(id), static_cast<uint32_t>(id >> 32), blk, 0u}, k0, k1);
      w[0] = o.x;
      w[1] = o.y;
      w[2] = o.z;
      w[3] = o.w;
    }
    bool exited = false;
    // The steps run unconditionally (predicated state updates, no per-step
    // branch).  A move onto an absorbing node (the halo around the lattice,
    // or a conductor voxel) is seen when that node's record id is loaded for
    // the next step; the walker then stops without consuming randomness.
    // The step cap is checked per super-step: a transit is an error iff it
    // needs more than `cap` steps (microwalk.cpp:81, :153-155), whichever
    // step inside the super-step crossed it.
#pragma unroll
    for (int u = 0; u < SS; ++u) {
      const uint32_t r = SMEM ? lds_u16(s_map + 2u * idx) : __ldg(g.map + idx);
      const bool act = live && !exited && r != kExit;
      exited |= live && r == kExit;
      uint64_t z = 0;
      uint32_t x11, h16 = 0;
      if (SM) {
        const uint64_t s1 = sm + kGamma;  // SplitMix64::next (rng.hpp:19-22)
        z = sm64_mix(s1);
        sm = act ? s1 : sm;
        x11 = static_cast<uint32_t>(z >> 53);  // top 11 bits of x = z >> 11
      } else {
        h16 = (u & 1) ? (w[u >> 1] & 0xFFFFu) : (w[u >> 1] >> 16);
        x11 = h16 >> 5;
      }
      steps += act;
      const uint64_t rc = SMEM ? lds_u64(s_rec + 8u * r) : __ldg(g.rec + r);
      // SWAR: lane d of x11*ones + rec = x11 + 2047 - T_d reaches its guard
      // bit iff x11 > T_d; the guard bits (11,23 | 35,47,59) of the low and
      // high words are disjoint, so one POPC of their OR counts them.  A lane
      // whose low 11 bits are all ones has x11 == T_d: a tie.
      const uint64_t d1 = static_cast<uint64_t>(x11) * kOnes + rc;
      const uint32_t lo = static_cast<uint32_t>(d1), hi = static_cast<uint32_t>(d1 >> 32);
      int dir = __popc((lo & static_cast<uint32_t>(kGuard)) |
                       (hi & static_cast<uint32_t>(kGuard >> 32)));
      const uint64_t d2 = d1 + kOnes;
      const bool tie = ((d2 ^ d1) & kGuard) != 0;
      if (__builtin_expect(__any_sync(0xFFFFFFFFu, act && tie), 0) && act && tie) {
        // 11-bit tie: exact comparison against the 53-bit thresholds
        const uint64_t* f = g.full + 5 * r;
        if (SM) {
          const uint64_t x53 = z >> 11;
          dir = 0;
#pragma unroll
          for (int d = 0; d < 5; ++d) dir += x53 >= __ldg(f + d);
        } else {
          dir = 0;
          bool tie16 = false;
#pragma unroll
          for (int d = 0; d < 5; ++d) {
            const uint64_t th = __ldg(f + d) >> 37;
            dir += h16 > th;
            tie16 |= h16 == th;
          }
          if (tie16) {
            const uint64_t id = static_cast<uint64_t>(p.stream_begin + t);
            const U32x4 o = philox4x32_10({static_cast<uint32_t>(id),
                                           static_cast<uint32_t>(id >> 32), blk * SS + u, 1u},
                                          k0, k1);
            const uint64_t low37 = ((static_cast<uint64_t>(o.x) << 32) | o.y) >> 27;
            const uint64_t x53 = (static_cast<uint64_t>(h16) << 37) | low37;
            dir = 0;
#pragma unroll
            for (int d = 0; d < 5; ++d) dir += x53 >= __ldg(f + d);
          }
        }
      }
      const int s = SMEM ? lds_s32(s_str + 4u * dir) : stride[dir];
      xdir = act ? dir : xdir;
      idx += act ? s : 0;
    }
    // the last step of the super-step may have moved onto an absorbing node
    {
      const uint32_t r = SMEM ? lds_u16(s_map + 2u * idx) : __ldg(g.map + idx);
      exited |= live && r == kExit;
    }
    ++blk;
    // ---- exit bookkeeping, batched once per super-step -------------------
    if (live && (exited || steps >= cap)) {
      int32_t panel = -1, cid = -1;
      long long nd = -1;
      if (exited && steps <= cap) {
        // absorbing node (padded coordinates) and the interior node before it
        const int hk = fdiv(idx, g.npp, g.inv_npp);
        const int hrem = idx - hk * g.npp;
        const int hj = fdiv(hrem, g.np, g.inv_np);
        const int hc[3] = {hrem - hj * g.np, hj, hk};
        const int ax = xdir >> 1;
        int c[3] = {hc[0] - 1, hc[1] - 1, hc[2] - 1};  // unpadded
        c[ax] -= (xdir & 1) ? 1 : -1;                  // step back inside
        nd = 8ll * ((c[2] * n + c[1]) * n + c[0]) + xdir;
        if (hc[ax] == 0 || hc[ax] == n + 1) {  // left the lattice: surface
          const int uu = ax == 0 ? c[1] : c[0];
          const int vv = ax == 2 ? c[1] : c[2];
          panel = (xdir * n + vv) * n + uu;  // sgf.hpp:34-36, sgf.cpp:13-30
          atomicAdd(hist + panel, 1ull);
        } else {  // absorbed by a conductor voxel (masked lattices)
          cid = g.mask[((hc[2] - 1) * n + (hc[1] - 1)) * n + (hc[0] - 1)];
          ++cexit;
        }
      } else {
        atomicExch(err, FRW_ESTEPCAP);  // microwalk.cpp:153-155
      }
      if (out_panel) out_panel[t] = panel;
      if (out_steps) out_steps[t] = steps;
      if (out_cond) out_cond[t] = cid;
      if (out_nd) out_nd[t] = nd;
      ssum += steps;
      ssq += static_cast<unsigned long long>(steps) * steps;
      // re-arm with the prefetched transit, prefetch the following one
      t = t_next;
      live = t < p.count;
      if (live) {
        t_next = static_cast<long long>(atomicAdd(ctr, 1ull));
        idx = g.start_idx;
        steps = 0;
        blk = 0;
        if (RNG == FRW_RNG_SPLITMIX_PARITY)
          sm = sm64_stream_from_mixed(p.mixed_seed, p.stream_begin + t);
        if (RNG == FRW_RNG_SPLITMIX_STATES) sm = p.states[t];
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ssum += __shfl_xor_sync(0xFFFFFFFFu, ssum, o);
    ssq += __shfl_xor_sync(0xFFFFFFFFu, ssq, o);
    cexit += __shfl_xor_sync(0xFFFFFFFFu, cexit, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(m_sum, ssum);
    atomicAdd(m_sq, ssq);
    atomicAdd(m_cx, cexit);
  }
}

// ---------------------------------------------------------------------------
// Fast path (table resident in shared memory, every record address < 64 KB):
//  * the staged node map holds each node's record as its shared-window byte
//    address, so a step is LDS.U16 -> LDS.64 with no address arithmetic, and
//    the walker's position is kept as the byte address of its map entry;
//  * the exit record is kGuard | 1<<63: every guard bit plus a sixth
//    counted bit, so an absorbed walker (and a retired lane parked on a halo
//    node) draws direction 6, whose stride is 0 -- no per-step predicates
//    on the move;
//  * tie test on one lane: with monotone thresholds the lanes whose guard
//    fired are exactly 0..dir-1, so x11 ties a threshold iff lane `dir` of
//    x11*ones + rec reads 2047 (its low 11 bits all ones);
//  * the step count is rebuilt at the super-step boundary from the index of
//    the last real step (steps = SS*blk + u_last + 1), so the loop carries
//    one predicated write per step instead of counter/select updates.

// low 32 bits of v >> s for 0 <= s <= 72 (PTX clamps shifts past 64 to 0)
__device__ __forceinline__ uint32_t shr64_lo(uint64_t v, uint32_t s) {
  uint32_t r;
  asm("{ .reg .b64 t; shr.b64 t, %1, %2; cvt.u32.u64 %0, t; }" : "=r"(r) : "l"(v), "r"(s));
  return r;
}

// Stage two segments into shared memory on one mbarrier.
__device__ void bulk_stage2(void* d0, const void* s0, uint32_t b0, void* d1, const void* s1,
                            uint32_t b1, uint64_t* bar) {
  const uint32_t b = smem_u32(bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(b0 + b1)
                 : "memory");
    constexpr uint32_t kChunk = 32768;
    for (int seg = 0; seg < 2; ++seg) {
      char* dst = static_cast<char*>(seg ? d1 : d0);
      const char* src = static_cast<const char*>(seg ? s1 : s0);
      const uint32_t bytes = seg ? b1 : b0;
      for (uint32_t off = 0; off < bytes; off += kChunk) {
        const uint32_t sz = min(kChunk, bytes - off);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
            "[%0], [%1], %2, [%3];" ::"r"(smem_u32(dst + off)),
            "l"(src + off), "r"(sz), "r"(b)
            : "memory");
      }
    }
  }
  __syncthreads();
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(b)
        : "memory");
  }
}

template <int RNG, bool TRACK>
__global__ void __launch_bounds__(kThreads, 1)
    mw_grid_fast(DevGrid g, DevParams p, unsigned long long* ctr, int* err,
                 int32_t* out_panel, int32_t* out_steps, int32_t* out_cond,
                 long long* out_nd, unsigned long long* hist, unsigned long long* m_sum,
                 unsigned long long* m_sq, unsigned long long* m_cx) {
  // TRACK: keep the direction of the last real step (for exit_nd); otherwise
  // the step count comes from a dwell counter and the exit panel from the
  // absorbing node alone (exit_info)
  constexpr bool SM = RNG != FRW_RNG_PHILOX;
  // Philox: FRW_GRID_PB blocks of 8 steps per super-step (the stream is the
  // same: block b of a transit is counter (id, b))
  constexpr int PB = SM ? 1 : FRW_GRID_PB;
  constexpr int SS = SM ? 4 : 8 * PB;
  // shared: records | node map | stride table (8 x s32) | mbarrier
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* rec_p = smem;
  uint8_t* map_p = smem + g.rec_bytes;
  int* str_p = reinterpret_cast<int*>(map_p + g.map_bytes);
  uint64_t* bar = reinterpret_cast<uint64_t*>(str_p + 8);
  bulk_stage2(rec_p, g.rec, g.rec_bytes, map_p, g.map, g.map_bytes, bar);
  const uint32_t s_rec = smem_base(rec_p);
  if (s_rec + g.rec_bytes > 65536u) {  // host guarantees this; never silently wrong
    if (threadIdx.x == 0) atomicExch(err, FRW_EINVAL);
    return;
  }
  // record ids -> record byte addresses, in place (two entries per word)
  for (uint32_t i = threadIdx.x; i < g.map_bytes / 4; i += kThreads) {
    uint32_t* w = reinterpret_cast<uint32_t*>(map_p) + i;
    const uint32_t v = *w;
    *w = (s_rec + 8u * (v & 0xFFFFu)) | ((s_rec + 8u * (v >> 16)) << 16);
  }
  if (threadIdx.x < 8) {
    const int d = threadIdx.x, ax = d >> 1;
    str_p[d] = d >= 6 ? 0 : ((d & 1) ? 2 : -2) * (ax == 0 ? 1 : ax == 1 ? g.np : g.npp);
  }
  __syncthreads();
  const uint32_t s_map = smem_base(map_p);
#if FRW_STRIDE_SHFL == 2
  // stride magnitudes as 16-bit fields {2, 2np, 2npp, 0}, selected by PRMT
  const uint32_t mag_lo = 2u | (static_cast<uint32_t>(2 * g.np) << 16);
  const uint32_t mag_hi = static_cast<uint32_t>(2 * g.npp);
#elif FRW_STRIDE_SHFL
  const int lane_stride = str_p[threadIdx.x & 7];
#else
  const uint32_t s_str = smem_base(str_p);
#endif
  // byte stride of direction d in the padded map (d = 6: the exit record's
  // stand-still)
  auto stride_of = [&](int d) -> uint32_t {
#if FRW_STRIDE_SHFL == 2
    // field d>>1 (upper bytes from the zero field 3), negated for even d: no
    // MIO op on the step's critical path
    uint32_t mag;
    asm("prmt.b32 %0, %1, %2, %3;"
        : "=r"(mag)
        : "r"(mag_lo), "r"(mag_hi), "r"(static_cast<uint32_t>(d & 6) * 0x11u + 0x7710u));
    return mag * static_cast<uint32_t>(2 * (d & 1) - 1);
#elif FRW_STRIDE_SHFL
    return static_cast<uint32_t>(__shfl_sync(0xFFFFFFFFu, lane_stride, d));
#else
    return static_cast<uint32_t>(lds_s32(s_str + 4u * d));
#endif
  };
  const uint32_t s_exit = s_rec + 8u * g.exit_rec;
  const uint32_t a_start = s_map + 2u * g.start_idx;
  const uint32_t ra_start = lds_u16(a_start);
  const uint32_t a_dead = s_map;  // padded node 0: a halo corner, absorbing

  const int n = g.n;
  const int cap = p.step_cap;
  unsigned long long ssum = 0, ssq = 0, cexit = 0;

  long long t = static_cast<long long>(atomicAdd(ctr, 1ull));
  long long t_next = static_cast<long long>(atomicAdd(ctr, 1ull));
  bool live = t < p.count;
  uint32_t a = live ? a_start : a_dead;
  uint32_t ra = live ? ra_start : s_exit;  // record address of the node at a
  uint32_t xinfo = 0;  // TRACK: (u << 3) | dir of the last real step
  int dwell = 0;       // !TRACK: steps drawn on an absorbing node this transit
  int blk = 0;         // super-steps completed in the current transit
  uint64_t sm = 0;
  if (RNG == FRW_RNG_SPLITMIX_PARITY && live)
    sm = sm64_stream_from_mixed(p.mixed_seed, p.stream_begin + t);
  if (RNG == FRW_RNG_SPLITMIX_STATES && live) sm = p.states[t];
  const uint32_t k0 = static_cast<uint32_t>(p.seed);
  const uint32_t k1 = static_cast<uint32_t>(p.seed >> 32);

  while (__any_sync(0xFFFFFFFFu, live)) {
    uint32_t w[4 * PB];
    if (RNG == FRW_RNG_PHILOX) {
      // one 4x32-10 call per 8 steps: word k gives step 2k its x11 from bits
      // 31..21 (16-bit prefix 31..16) and step 2k+1 from bits 10..0 (prefix
      // continues with bits 15..11); the low 37 bits of x come from the
      // (id, step slot, 1) counter only on a 16-bit tie
      const uint64_t id = static_cast<uint64_t>(p.stream_begin + t);
#pragma unroll
      for (int c = 0; c < PB; ++c) {
        const U32x4 o = philox4x32_10(
            {static_cast<uint32_t>(id), static_cast<uint32_t>(id >> 32),
             static_cast<uint32_t>(blk * PB + c), 0u},
            k0, k1);
        w[4 * c] = o.x;
        w[4 * c + 1] = o.y;
        w[4 * c + 2] = o.z;
        w[4 * c + 3] = o.w;
      }
    }
#pragma unroll
    for (int u = 0; u < SS; ++u) {
      const bool act = ra != s_exit;
      const uint64_t rc = lds_u64(ra);
      uint64_t z = 0;
      uint32_t x11;
      if (SM) {
        const uint64_t s1 = sm + kGamma;  // SplitMix64::next (rng.hpp:19-22)
        z = sm64_mix(s1);
        if (act) sm = s1;  // an absorbed walker consumes no randomness
        x11 = static_cast<uint32_t>(z >> 53);
      } else {
        x11 = (u & 1) ? (w[u >> 1] & 0x7FFu) : (w[u >> 1] >> 21);
      }
      const uint64_t d1 = static_cast<uint64_t>(x11) * kOnes + rc;
      const uint32_t d1h = static_cast<uint32_t>(d1 >> 32);
      int dir = __popc((static_cast<uint32_t>(d1) & kGuardLo) | (d1h & kGuardHi));
      // (absorbed lanes never tie: their shift is 72, which PTX clamps to 0)
      const bool tie = (~shr64_lo(d1, 12u * dir) & 0x7FFu) == 0;
      // move first (the common case) so the next map load is in flight while
      // the tie test resolves; a tied lane redoes its move in the tie block
      const uint32_t a0 = a, ra0 = ra;
      a = a0 + stride_of(dir);
      ra = lds_u16(a);
      if (__builtin_expect(__any_sync(0xFFFFFFFFu, tie), 0)) {
        // 11-bit tie: exact comparison against the 53-bit thresholds.  The
        // block is warp-uniform (predicated per lane), so the common path
        // carries no reconvergence barrier.
        const uint64_t* f = g.full + 5 * ((ra0 - s_rec) >> 3);
        uint64_t th[5];
#pragma unroll
        for (int d = 0; d < 5; ++d) th[d] = tie ? __ldg(f + d) : 0;
        int dx = 0;
        if (SM) {
          const uint64_t x53 = z >> 11;
#pragma unroll
          for (int d = 0; d < 5; ++d) dx += x53 >= th[d];
        } else {
          const uint32_t wu = w[u >> 1];
          const uint32_t h16 =
              (u & 1) ? (((wu & 0x7FFu) << 5) | ((wu >> 11) & 0x1Fu)) : (wu >> 16);
          bool tie16 = false;
#pragma unroll
          for (int d = 0; d < 5; ++d) {
            const uint32_t t16 = static_cast<uint32_t>(th[d] >> 37);
            dx += h16 > t16;
            tie16 |= h16 == t16;
          }
          tie16 = tie16 && tie;
          if (__any_sync(0xFFFFFFFFu, tie16)) {
            const uint64_t id = static_cast<uint64_t>(p.stream_begin + t);
            const U32x4 o = philox4x32_10(
                {static_cast<uint32_t>(id), static_cast<uint32_t>(id >> 32),
                 static_cast<uint32_t>(blk * SS + u), 1u},
                k0, k1);
            const uint64_t low37 = ((static_cast<uint64_t>(o.x) << 32) | o.y) >> 27;
            const uint64_t x53 = (static_cast<uint64_t>(h16) << 37) | low37;
            int de = 0;
#pragma unroll
            for (int d = 0; d < 5; ++d) de += x53 >= th[d];
            dx = tie16 ? de : dx;
          }
        }
        dir = tie ? dx : dir;
        const uint32_t a1 = a0 + stride_of(dir);  // (all lanes: the shuffle)
        if (tie) {
          a = a1;
          ra = lds_u16(a1);
        }
      }
      if (TRACK) {
        if (act) xinfo = (u << 3) | dir;
      } else {
        dwell += d1h >> 31;  // the exit record's bit 63 survives the add
      }
    }
    // ---- exit bookkeeping, once per super-step ---------------------------
    const bool exited = ra == s_exit;
    const int steps = TRACK ? (exited ? SS * blk + static_cast<int>(xinfo >> 3) + 1 : SS * (blk + 1))
                            : SS * (blk + 1) - dwell;
    ++blk;
    if (live && (exited || steps >= cap)) {
      int32_t panel = -1, cid = -1;
      long long nd = -1;
      if (exited && steps <= cap) {
        const int idx = static_cast<int>((a - s_map) >> 1);
        const int info = __ldg(g.exit_info + idx);
        if (info >= 0) {  // left the lattice: surface panel
          panel = info;
          atomicAdd(hist + panel, 1ull);
        } else {  // absorbed by a conductor voxel (masked lattices)
          cid = -2 - info;
          ++cexit;
        }
        if (TRACK) {  // the interior node before the exit and the direction
          const int xdir = static_cast<int>(xinfo & 7u);
          const int hk = fdiv(idx, g.npp, g.inv_npp);
          const int hrem = idx - hk * g.npp;
          const int hj = fdiv(hrem, g.np, g.inv_np);
          int c[3] = {hrem - hj * g.np - 1, hj - 1, hk - 1};  // unpadded
          const int ax = xdir >> 1;
          c[ax] -= (xdir & 1) ? 1 : -1;  // step back inside
          nd = 8ll * ((c[2] * n + c[1]) * n + c[0]) + xdir;
        }
      } else {
        atomicExch(err, FRW_ESTEPCAP);  // microwalk.cpp:153-155
      }
      if (out_panel) out_panel[t] = panel;
      if (out_steps) out_steps[t] = steps;
      if (out_cond) out_cond[t] = cid;
      if (out_nd) out_nd[t] = nd;
      ssum += steps;
      ssq += static_cast<unsigned long long>(steps) * steps;
      // re-arm with the prefetched transit, prefetch the following one
      t = t_next;
      live = t < p.count;
      blk = 0;
      dwell = 0;
      a = live ? a_start : a_dead;
      ra = live ? ra_start : s_exit;
      if (live) {
        t_next = static_cast<long long>(atomicAdd(ctr, 1ull));
        if (RNG == FRW_RNG_SPLITMIX_PARITY)
          sm = sm64_stream_from_mixed(p.mixed_seed, p.stream_begin + t);
        if (RNG == FRW_RNG_SPLITMIX_STATES) sm = p.states[t];
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ssum += __shfl_xor_sync(0xFFFFFFFFu, ssum, o);
    ssq += __shfl_xor_sync(0xFFFFFFFFu, ssq, o);
    cexit += __shfl_xor_sync(0xFFFFFFFFu, cexit, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(m_sum, ssum);
    atomicAdd(m_sq, ssq);
    atomicAdd(m_cx, cexit);
  }
}

template <int RNG, bool SMEM>
int launch(frw_ctx* ctx, const frw_mw_params* p, const frw_mw_out* o, unsigned long long* ms,
           unsigned long long* mq, unsigned long long* mc) {
  const GridTable& G = ctx->grid;
  const int np = G.n + 2;
  DevGrid g{G.d_map, G.d_rec, G.d_full, G.has_mask ? G.d_mask : nullptr, G.d_exit, G.n, np, np * np,
            G.start_idx, static_cast<uint32_t>(G.records),
            static_cast<uint32_t>(G.map_bytes), static_cast<uint32_t>(G.rec_bytes),
            1.0f / np, 1.0f / (np * np)};
  DevParams dp{p->seed, sm64_mix(p->seed), p->stream_begin, p->count,
               p->step_cap > 0 ? p->step_cap : 1000 * G.n * G.n, p->states};
  // fast path: records addressable by 16-bit shared addresses (the window
  // base is at most a few KB; the kernel checks the exact bound)
  const bool fast = SMEM && G.rec_bytes + 4096 <= 65536;
  const size_t smem = !SMEM ? 0 : fast ? G.map_bytes + G.rec_bytes + 48 : G.map_bytes + G.rec_bytes;
  auto kern = !fast ? mw_grid_kernel<RNG, SMEM>
              : o->exit_nd ? mw_grid_fast<RNG, true> : mw_grid_fast<RNG, false>;
  if (SMEM)
    FRW_CUDA(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem)));
  FRW_CUDA(ctx, cudaMemsetAsync(ctx->d_ctr, 0, sizeof(unsigned long long), ctx->stream));
  const int blocks = p->blocks > 0 ? p->blocks : ctx->sm_count;
  kern<<<blocks, kThreads, smem, ctx->stream>>>(
      g, dp, ctx->d_ctr, ctx->d_err, o->panels, o->steps, o->cond,
      reinterpret_cast<long long*>(o->exit_nd), reinterpret_cast<unsigned long long*>(o->hist),
      ms, mq, mc);
  FRW_CUDA(ctx, cudaGetLastError());
  return FRW_OK;
}


// ---------------------------------------------------------------------------
// On-device compile of the cube (the e2e path: only the permittivities cross
// PCIe).  The same records as compile_grid -- alphas en / (en + ev), their
// in-order partial sums and the exact thresholds of threshold_of, all plain
// IEEE f64 -- numbered in whatever order the hash inserts land (the record
// numbering is invisible to the walk: a node's record content is what it
// steps with, and the exact thresholds follow the record).  A stencil key is
// the node's palette id and its six neighbour codes at 9 bits each, so
// palettes of up to kDcPal permittivities compile here; larger ones (and
// FRW_GRID_HOST_COMPILE=1) take compile_grid.
constexpr uint32_t kDcPal = 510;           // palette ids; 510 = conductor, 511 = surface
constexpr uint32_t kDcCond = 510, kDcSurf = 511;

struct DcBufs {
  double* eps;          // [n^3] staged permittivities
  int32_t* mask;        // [n^3] or null
  uint64_t* pal_key;    // [pcap] eps bits (0: empty)
  uint32_t* pal_val;    // [pcap]
  double* pal_eps;      // [kDcPal]
  uint64_t* rec_key;    // [rcap] stencil keys (0: empty)
  uint32_t* rec_val;    // [rcap]
  uint64_t* rec_of;     // [kRecMax] key of record r
  uint32_t* node_pal;   // [n^3]
  uint32_t* cnt;        // [0] palette size, [1] records, [2] error
  uint32_t pmask, rmask;
};
constexpr uint32_t kRecMax = 65535;

__device__ __forceinline__ uint32_t dc_hash(uint64_t k) { return static_cast<uint32_t>(sm64_mix(k)); }

__global__ void k_dc_palette(int nodes, DcBufs B) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nodes; v += gridDim.x * blockDim.x) {
    const double e = B.eps[v];
    if (!(e > 0) || !isfinite(e)) {
      atomicMax(&B.cnt[2], 1u);
      continue;
    }
    const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(e));
    for (uint32_t h = dc_hash(bits) & B.pmask;; h = (h + 1) & B.pmask) {
      const unsigned long long prev = atomicCAS(reinterpret_cast<unsigned long long*>(B.pal_key + h), 0ull,
                                                static_cast<unsigned long long>(bits));
      if (prev == 0) {
        const uint32_t id = atomicAdd(&B.cnt[0], 1u);
        B.pal_val[h] = id;
        if (id < kDcPal) B.pal_eps[id] = e;
        break;
      }
      if (prev == bits) break;
    }
  }
}

__global__ void k_dc_node_pal(int nodes, DcBufs B) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nodes; v += gridDim.x * blockDim.x) {
    const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(B.eps[v]));
    uint32_t h = dc_hash(bits) & B.pmask;
    while (B.pal_key[h] != bits) h = (h + 1) & B.pmask;
    B.node_pal[v] = B.pal_val[h];
  }
}

// the stencil key of lattice node (i, j, k): its palette id and the six
// neighbour codes (surface / conductor / palette id), 9 bits each; bit 63 set
__device__ __forceinline__ uint64_t dc_key(const DcBufs& B, int n, int i, int j, int k) {
  const int v = (k * n + j) * n + i;
  const uint32_t self = B.node_pal[v];
  uint64_t key = (1ull << 63) | self;
  bool uniform = true;  // every non-absorbing neighbour has the node's permittivity
#pragma unroll
  for (int d = 0; d < 6; ++d) {
    int nb[3] = {i, j, k};
    nb[d >> 1] += (d & 1) ? 1 : -1;
    uint32_t code;
    if (nb[d >> 1] < 0 || nb[d >> 1] >= n) {
      code = kDcSurf;
    } else {
      const int nv = (nb[2] * n + nb[1]) * n + nb[0];
      code = (B.mask && B.mask[nv] >= 0) ? kDcCond : B.node_pal[nv];
    }
    uniform = uniform && (code == self || code >= kDcCond);
    key |= static_cast<uint64_t>(code) << (9 * (d + 1));
  }
  // all alphas 1/2 or 1 whatever the permittivity: palette id 0 stands for it
  // (see compile_grid), one record for every uniform neighbourhood
  if (uniform && self < kDcPal && same_eps_halves(B.pal_eps[self]) && same_eps_halves(B.pal_eps[0])) {
    uint64_t canon = 1ull << 63;
#pragma unroll
    for (int d = 0; d < 6; ++d) {
      const uint64_t code = (key >> (9 * (d + 1))) & 0x1FF;
      canon |= (code >= kDcCond ? code : 0ull) << (9 * (d + 1));
    }
    key = canon;
  }
  return key;
}

__global__ void k_dc_records(int n, DcBufs B) {
  const int nodes = n * n * n;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nodes; v += gridDim.x * blockDim.x) {
    if (B.mask && B.mask[v] >= 0) continue;  // conductor voxel: the exit record
    const uint64_t key = dc_key(B, n, v % n, (v / n) % n, v / (n * n));
    for (uint32_t h = dc_hash(key) & B.rmask;; h = (h + 1) & B.rmask) {
      const unsigned long long prev = atomicCAS(reinterpret_cast<unsigned long long*>(B.rec_key + h), 0ull,
                                                static_cast<unsigned long long>(key));
      if (prev == 0) {
        const uint32_t r = atomicAdd(&B.cnt[1], 1u);
        B.rec_val[h] = r;
        if (r < kRecMax) B.rec_of[r] = key;
        break;
      }
      if (prev == key) break;
    }
  }
}

// padded map: record id of each lattice node, the exit record (id R) on the
// halo and on conductor voxels
__global__ void k_dc_map(int n, DcBufs B, uint16_t* map) {
  const int np = n + 2, total = np * np * np;
  const uint32_t R = B.cnt[1];
  for (int pv = blockIdx.x * blockDim.x + threadIdx.x; pv < total; pv += gridDim.x * blockDim.x) {
    const int i = pv % np - 1, j = (pv / np) % np - 1, k = pv / (np * np) - 1;
    uint32_t r = R;
    if (i >= 0 && i < n && j >= 0 && j < n && k >= 0 && k < n &&
        !(B.mask && B.mask[(k * n + j) * n + i] >= 0)) {
      const uint64_t key = dc_key(B, n, i, j, k);
      uint32_t h = dc_hash(key) & B.rmask;
      while (B.rec_key[h] != key) h = (h + 1) & B.rmask;
      r = B.rec_val[h];
    }
    map[pv] = static_cast<uint16_t>(r);
  }
}

// record contents (microwalk.cpp:91-109 alphas, exact thresholds), then the exit record
__global__ void k_dc_contents(DcBufs B, uint64_t* rec, uint64_t* full) {
  const uint32_t R = B.cnt[1];
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r <= R; r += gridDim.x * blockDim.x) {
    if (r == R) {
      rec[R] = kExitRec;
      for (int d = 0; d < 5; ++d) full[5ull * R + d] = 1ull << 53;
      continue;
    }
    const uint64_t key = B.rec_of[r];
    const double ev = B.pal_eps[key & 0x1FF];
    double acc[6], sum = 0;
#pragma unroll
    for (int d = 0; d < 6; ++d) {
      const uint32_t code = static_cast<uint32_t>(key >> (9 * (d + 1))) & 0x1FF;
      double a = 1.0;
      if (code < kDcCond) {
        const double en = B.pal_eps[code];
        a = en / (en + ev);
      }
      sum += a;
      acc[d] = sum;
    }
    uint64_t packed = 0;
#pragma unroll
    for (int d = 0; d < 5; ++d) {
      const uint64_t X = threshold_of(acc[d], sum);
      full[5ull * r + d] = X;
      const uint64_t t11 = X >> 42 < static_cast<uint64_t>(kTop) ? X >> 42 : kTop;
      packed |= (kTop - t11) << (kLane * d);
    }
    rec[r] = packed;
  }
}

// exit_info_of on the device (see there)
__global__ void k_dc_exit(int n, const int32_t* mask, int32_t* info) {
  const int np = n + 2, total = np * np * np;
  for (int pv = blockIdx.x * blockDim.x + threadIdx.x; pv < total; pv += gridDim.x * blockDim.x) {
    const int h[3] = {pv % np, (pv / np) % np, pv / (np * np)};
    int out = 0, ax = -1;
#pragma unroll
    for (int a = 0; a < 3; ++a)
      if (h[a] == 0 || h[a] == n + 1) ++out, ax = a;
    int r = -1;
    if (out == 0) {
      if (mask) {
        const int m = mask[((h[2] - 1) * n + (h[1] - 1)) * n + (h[0] - 1)];
        if (m >= 0) r = -2 - m;
      }
    } else if (out == 1) {
      const int dir = 2 * ax + (h[ax] == n + 1 ? 1 : 0);
      int c[3] = {h[0] - 1, h[1] - 1, h[2] - 1};
      c[ax] = h[ax] == 0 ? 0 : n - 1;
      const int uu = ax == 0 ? c[1] : c[0];
      const int vv = ax == 2 ? c[1] : c[2];
      r = (dir * n + vv) * n + uu;
    }
    info[pv] = r;
  }
}


inline size_t pow2_at_least(size_t v) {
  size_t c = 1024;
  while (c < v) c <<= 1;
  return c;
}

// The device compile driver (see k_dc_*): stages eps (and the mask), builds
// palette and stencil tables, then map, records, exact thresholds and the
// exit table straight into the GridTable buffers.  Returns 1 when the grid
// needs the host compile (palette past kDcPal), FRW_OK, or an error.
int compile_grid_device(frw_ctx* ctx, int n, const double* eps, const int32_t* mask) {
  GridTable& G = ctx->grid;
  const size_t nodes = static_cast<size_t>(n) * n * n;
  const int np = n + 2;
  const size_t pnodes = static_cast<size_t>(np) * np * np;
  const size_t pcap = pow2_at_least(2 * nodes), rcap = pow2_at_least(2 * std::min<size_t>(nodes, kRecMax));
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  const size_t o_eps = 0, o_mask = o_eps + al(8 * nodes), o_pk = o_mask + (mask ? al(4 * nodes) : 0),
               o_pv = o_pk + al(8 * pcap), o_pe = o_pv + al(4 * pcap), o_rk = o_pe + al(8 * 512),
               o_rv = o_rk + al(8 * rcap), o_ro = o_rv + al(4 * rcap), o_np = o_ro + al(8 * kRecMax),
               o_cnt = o_np + al(4 * nodes), need = o_cnt + 256;
  if (G.dc_cap < need) {
    cudaFree(G.d_dc);
    G.d_dc = nullptr;
    G.dc_cap = 0;
    FRW_CUDA(ctx, cudaMalloc(&G.d_dc, need));
    G.dc_cap = need;
  }
  char* b = G.d_dc;
  DcBufs B{reinterpret_cast<double*>(b + o_eps),
           mask ? reinterpret_cast<int32_t*>(b + o_mask) : nullptr,
           reinterpret_cast<uint64_t*>(b + o_pk), reinterpret_cast<uint32_t*>(b + o_pv),
           reinterpret_cast<double*>(b + o_pe), reinterpret_cast<uint64_t*>(b + o_rk),
           reinterpret_cast<uint32_t*>(b + o_rv), reinterpret_cast<uint64_t*>(b + o_ro),
           reinterpret_cast<uint32_t*>(b + o_np), reinterpret_cast<uint32_t*>(b + o_cnt),
           static_cast<uint32_t>(pcap - 1), static_cast<uint32_t>(rcap - 1)};
  cudaStream_t st = ctx->stream;
  FRW_CUDA(ctx, cudaMemcpyAsync(B.eps, eps, 8 * nodes, cudaMemcpyHostToDevice, st));
  if (mask) FRW_CUDA(ctx, cudaMemcpyAsync(B.mask, mask, 4 * nodes, cudaMemcpyHostToDevice, st));
  FRW_CUDA(ctx, cudaMemsetAsync(B.pal_key, 0, 8 * pcap, st));
  FRW_CUDA(ctx, cudaMemsetAsync(B.rec_key, 0, 8 * rcap, st));
  FRW_CUDA(ctx, cudaMemsetAsync(B.cnt, 0, 16, st));
  const int grid = ctx->sm_count * 4;
  k_dc_palette<<<grid, 256, 0, st>>>(static_cast<int>(nodes), B);
  k_dc_node_pal<<<grid, 256, 0, st>>>(static_cast<int>(nodes), B);
  k_dc_records<<<grid, 256, 0, st>>>(n, B);
  uint32_t cnt[3] = {0, 0, 0};
  FRW_CUDA(ctx, cudaMemcpyAsync(cnt, B.cnt, 12, cudaMemcpyDeviceToHost, st));
  FRW_CUDA(ctx, cudaStreamSynchronize(st));
  if (cnt[2]) return frw_fail(ctx, FRW_EINVAL, "grid permittivities must be finite and > 0");
  if (cnt[0] > kDcPal) return 1;  // palette past the 9-bit key fields: host compile
  if (cnt[1] >= kRecMax)
    return frw_fail(ctx, FRW_EINVAL, "more than 65535 distinct stencil records");
  const uint32_t R = cnt[1];
  G.n = n;
  G.records = static_cast<int>(R);
  G.map_bytes = (pnodes * 2 + 15) / 16 * 16;
  G.rec_bytes = ((R + 1) * 8 + 15) / 16 * 16;
  const size_t blob = G.map_bytes + G.rec_bytes, full = (R + 1) * 5 * 8;
  if (G.blob_cap < blob) {
    cudaFree(G.d_map);
    G.d_map = nullptr;
    G.blob_cap = 0;
    char* p = nullptr;
    FRW_CUDA(ctx, cudaMalloc(&p, blob));
    G.d_map = reinterpret_cast<uint16_t*>(p);
    G.blob_cap = blob;
  }
  G.d_rec = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(G.d_map) + G.map_bytes);
  if (G.full_cap < full) {
    cudaFree(G.d_full);
    G.d_full = nullptr;
    G.full_cap = 0;
    FRW_CUDA(ctx, cudaMalloc(&G.d_full, full));
    G.full_cap = full;
  }
  k_dc_map<<<grid, 256, 0, st>>>(n, B, G.d_map);
  k_dc_contents<<<(R + 256) / 256, 256, 0, st>>>(B, G.d_rec, G.d_full);
  if (mask || G.exit_n != n) {  // the exit table of an unmasked lattice depends on n only
    if (G.exit_cap < 4 * pnodes) {
      cudaFree(G.d_exit);
      G.d_exit = nullptr;
      G.exit_cap = 0;
      FRW_CUDA(ctx, cudaMalloc(&G.d_exit, 4 * pnodes));
      G.exit_cap = 4 * pnodes;
    }
    k_dc_exit<<<grid, 256, 0, st>>>(n, B.mask, G.d_exit);
    G.exit_n = mask ? 0 : n;
  }
  FRW_CUDA(ctx, cudaGetLastError());
  G.h2d_bytes = 8 * nodes + (mask ? 4 * nodes : 0);
  return FRW_OK;
}

}  // namespace
}  // namespace frw

using namespace frw;

extern "C" {

int frw_upload_grid(frw_ctx* ctx, int n, const double* eps, const int32_t* mask, double cx,
                    double cy, double cz, double half_width) {
  if (!ctx) return FRW_EINVAL;
  if (n < 1 || n > 253 || !eps)
    return frw_fail(ctx, FRW_EINVAL, "upload_grid: need 1 <= n <= 253 and eps");
  if (!(half_width > 0)) return frw_fail(ctx, FRW_EINVAL, "upload_grid: half_width <= 0");
  FRW_CUDA(ctx, cudaSetDevice(ctx->device));
  GridTable& G = ctx->grid;
  const int c = (n - 1) / 2;  // start_node, sgf.hpp:58-61
  const int np = n + 2;
  G.start_idx = ((c + 1) * np + (c + 1)) * np + (c + 1);  // padded
  G.start_is_conductor = mask && mask[(c * n + c) * n + c] >= 0;
  G.center[0] = cx;
  G.center[1] = cy;
  G.center[2] = cz;
  G.half_width = half_width;
  G.has_mask = mask != nullptr;
  if (mask) {  // the walk kernels read the mask of a masked lattice
    const size_t bytes = static_cast<size_t>(n) * n * n * 4;
    if (G.mask_cap < bytes) {
      cudaFree(G.d_mask);
      G.d_mask = nullptr;
      G.mask_cap = 0;
      FRW_CUDA(ctx, cudaMalloc(&G.d_mask, bytes));
      G.mask_cap = bytes;
    }
    FRW_CUDA(ctx, cudaMemcpyAsync(G.d_mask, mask, bytes, cudaMemcpyHostToDevice, ctx->stream));
  }
  // compile on the device (only eps crosses PCIe); FRW_GRID_HOST_COMPILE=1
  // or a palette past 510 permittivities compiles on the host
  static const bool host_only = [] {
    const char* e = std::getenv("FRW_GRID_HOST_COMPILE");
    return e && std::atoi(e) != 0;
  }();
  if (!host_only) {
    const int rc = compile_grid_device(ctx, n, eps, mask);
    if (rc == FRW_OK) {
      G.host_compiled = false;
      FRW_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
      return FRW_OK;
    }
    if (rc != 1) return rc;
  }
  G.host_compiled = true;
  G.exit_n = 0;
  Compiled cg;
  if (int rc = compile_grid(ctx, n, eps, mask, cg)) return rc;
  G.n = n;
  G.records = static_cast<int>(cg.rec.size()) - 1;  // step records; [R] is the exit record
  G.map_bytes = (cg.map.size() * 2 + 15) / 16 * 16;
  G.rec_bytes = (cg.rec.size() * 8 + 15) / 16 * 16;
  // one allocation: map then packed records, so one bulk stage covers both;
  // buffers are kept across uploads and grown only when too small
  const size_t blob = G.map_bytes + G.rec_bytes, full = cg.full.size() * 8;
  if (G.blob_cap < blob) {
    cudaFree(G.d_map);  // also releases d_rec (same allocation)
    G.d_map = nullptr;
    G.blob_cap = 0;
    char* p = nullptr;
    FRW_CUDA(ctx, cudaMalloc(&p, blob));
    G.d_map = reinterpret_cast<uint16_t*>(p);
    G.blob_cap = blob;
  }
  G.d_rec = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(G.d_map) + G.map_bytes);
  if (G.full_cap < full) {
    cudaFree(G.d_full);
    G.d_full = nullptr;
    G.full_cap = 0;
    FRW_CUDA(ctx, cudaMalloc(&G.d_full, full));
    G.full_cap = full;
  }
  FRW_CUDA(ctx, cudaMemcpyAsync(G.d_map, cg.map.data(), cg.map.size() * 2,
                                cudaMemcpyHostToDevice, ctx->stream));
  FRW_CUDA(ctx, cudaMemcpyAsync(G.d_rec, cg.rec.data(), cg.rec.size() * 8,
                                cudaMemcpyHostToDevice, ctx->stream));
  FRW_CUDA(ctx, cudaMemcpyAsync(G.d_full, cg.full.data(), full, cudaMemcpyHostToDevice,
                                ctx->stream));
  const size_t ebytes = cg.exit_info.size() * 4;
  if (G.exit_cap < ebytes) {
    cudaFree(G.d_exit);
    G.d_exit = nullptr;
    G.exit_cap = 0;
    FRW_CUDA(ctx, cudaMalloc(&G.d_exit, ebytes));
    G.exit_cap = ebytes;
  }
  FRW_CUDA(ctx, cudaMemcpyAsync(G.d_exit, cg.exit_info.data(), ebytes, cudaMemcpyHostToDevice,
                                ctx->stream));
  G.h2d_bytes = cg.map.size() * 2 + cg.rec.size() * 8 + full + ebytes +
                (mask ? static_cast<size_t>(n) * n * n * 4 : 0);
  FRW_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return FRW_OK;
}

int frw_grid_compile(int n, const double* eps, const int32_t* mask, uint16_t* map,
                     uint64_t* rec, uint64_t* full, int* records) {
  if (n < 1 || n > 253 || !eps || !records) return FRW_EINVAL;
  frw_ctx tmp;
  Compiled cg;
  if (int rc = compile_grid(&tmp, n, eps, mask, cg)) return rc;
  *records = static_cast<int>(cg.rec.size());
  if (map) std::memcpy(map, cg.map.data(), cg.map.size() * 2);
  if (rec) std::memcpy(rec, cg.rec.data(), cg.rec.size() * 8);
  if (full) std::memcpy(full, cg.full.data(), cg.full.size() * 8);
  return FRW_OK;
}

int frw_grid_info(const frw_ctx* ctx, int* records, int* smem_bytes, int* smem_resident) {
  if (!ctx) return FRW_EINVAL;
  const GridTable& G = ctx->grid;
  const size_t bytes = G.map_bytes + G.rec_bytes;
  if (records) *records = G.records;
  if (smem_bytes) *smem_bytes = static_cast<int>(bytes);
  if (smem_resident) *smem_resident = bytes + 1024 <= static_cast<size_t>(ctx->max_smem_optin);
  return FRW_OK;
}

int frw_grid_h2d_bytes(const frw_ctx* ctx, uint64_t* bytes) {
  if (!ctx || !bytes) return FRW_EINVAL;
  *bytes = ctx->grid.h2d_bytes;
  return FRW_OK;
}

int frw_microwalk_batch_dev(frw_ctx* ctx, const frw_mw_params* p, const frw_mw_out* o) {
  if (!ctx || !p || !o) return FRW_EINVAL;
  const GridTable& G = ctx->grid;
  if (!G.d_map) return frw_fail(ctx, FRW_EINVAL, "microwalk_batch: no grid uploaded");
  if (!o->hist) return frw_fail(ctx, FRW_EINVAL, "microwalk_batch: hist is required");
  if (p->count < 0) return frw_fail(ctx, FRW_EINVAL, "microwalk_batch: count < 0");
  if (G.start_is_conductor)
    return frw_fail(ctx, FRW_EENGULFED, "transit start voxel lies inside a conductor");
  if (p->rng_mode != FRW_RNG_SPLITMIX_PARITY && p->rng_mode != FRW_RNG_PHILOX &&
      p->rng_mode != FRW_RNG_SPLITMIX_STATES)
    return frw_fail(ctx, FRW_EINVAL, "microwalk_batch: unknown rng mode");
  if (p->rng_mode == FRW_RNG_SPLITMIX_STATES && !p->states)
    return frw_fail(ctx, FRW_EINVAL, "microwalk_batch: states required");
  FRW_CUDA(ctx, cudaSetDevice(ctx->device));
  if (p->count == 0) return FRW_OK;
  auto* ms = reinterpret_cast<unsigned long long*>(o->step_sum ? o->step_sum : ctx->d_mom);
  auto* mq = reinterpret_cast<unsigned long long*>(o->step_sumsq ? o->step_sumsq : ctx->d_mom + 1);
  auto* mc = reinterpret_cast<unsigned long long*>(o->cond_exits ? o->cond_exits : ctx->d_mom + 2);
  const bool smem = G.map_bytes + G.rec_bytes + 1024 <= static_cast<size_t>(ctx->max_smem_optin);
  if (p->rng_mode == FRW_RNG_SPLITMIX_PARITY)
    return smem ? launch<FRW_RNG_SPLITMIX_PARITY, true>(ctx, p, o, ms, mq, mc)
                : launch<FRW_RNG_SPLITMIX_PARITY, false>(ctx, p, o, ms, mq, mc);
  if (p->rng_mode == FRW_RNG_SPLITMIX_STATES)
    return smem ? launch<FRW_RNG_SPLITMIX_STATES, true>(ctx, p, o, ms, mq, mc)
                : launch<FRW_RNG_SPLITMIX_STATES, false>(ctx, p, o, ms, mq, mc);
  return smem ? launch<FRW_RNG_PHILOX, true>(ctx, p, o, ms, mq, mc)
              : launch<FRW_RNG_PHILOX, false>(ctx, p, o, ms, mq, mc);
}

int frw_microwalk_check(frw_ctx* ctx) {
  if (!ctx) return FRW_EINVAL;
  int flag = 0;
  FRW_CUDA(ctx, cudaMemcpyAsync(&flag, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost,
                                ctx->stream));
  FRW_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  FRW_CUDA(ctx, cudaMemsetAsync(ctx->d_err, 0, sizeof(int), ctx->stream));
  if (flag)
    return frw_fail(ctx, flag, "microwalk transit exceeded the step cap; the lattice is malformed");
  return FRW_OK;
}

int frw_microwalk_batch(frw_ctx* ctx, const frw_mw_params* p, const frw_mw_out* host) {
  if (!ctx || !p || !host) return FRW_EINVAL;
  const GridTable& G = ctx->grid;
  if (!G.d_map) return frw_fail(ctx, FRW_EINVAL, "microwalk_batch: no grid uploaded");
  FRW_CUDA(ctx, cudaSetDevice(ctx->device));
  const size_t bins = 6ull * G.n * G.n;
  if (ctx->hist_cap < bins) {
    cudaFree(ctx->d_hist);
    FRW_CUDA(ctx, cudaMalloc(&ctx->d_hist, bins * 8));
    ctx->hist_cap = bins;
  }
  // per-transit scratch: panels | steps | cond (int32) | exit_nd (int64) |
  // states (u64)
  const size_t cnt = static_cast<size_t>(std::max<int64_t>(p->count, 0));
  const bool states = p->rng_mode == FRW_RNG_SPLITMIX_STATES;
  const bool per = host->panels || host->steps || host->cond || host->exit_nd || states;
  const size_t off_nd = (12 * cnt + 7) / 8 * 8, off_st = off_nd + 8 * cnt, need = off_st + 8 * cnt;
  if (per && ctx->tr_cap < need) {
    cudaFree(ctx->d_tr);
    ctx->d_tr = nullptr;
    ctx->tr_cap = 0;
    FRW_CUDA(ctx, cudaMalloc(&ctx->d_tr, need));
    ctx->tr_cap = need;
  }
  char* tr = reinterpret_cast<char*>(ctx->d_tr);
  FRW_CUDA(ctx, cudaMemsetAsync(ctx->d_hist, 0, bins * 8, ctx->stream));
  FRW_CUDA(ctx, cudaMemsetAsync(ctx->d_mom, 0, 32, ctx->stream));
  FRW_CUDA(ctx, cudaMemsetAsync(ctx->d_err, 0, sizeof(int), ctx->stream));
  frw_mw_out d{};
  d.hist = ctx->d_hist;
  d.step_sum = ctx->d_mom;
  d.step_sumsq = ctx->d_mom + 1;
  d.cond_exits = ctx->d_mom + 2;
  if (host->panels) d.panels = reinterpret_cast<int32_t*>(tr);
  if (host->steps) d.steps = reinterpret_cast<int32_t*>(tr) + cnt;
  if (host->cond) d.cond = reinterpret_cast<int32_t*>(tr) + 2 * cnt;
  if (host->exit_nd) d.exit_nd = reinterpret_cast<int64_t*>(tr + off_nd);
  frw_mw_params pd = *p;
  if (states) {
    if (!p->states) return frw_fail(ctx, FRW_EINVAL, "microwalk_batch: states required");
    FRW_CUDA(ctx, cudaMemcpyAsync(tr + off_st, p->states, 8 * cnt, cudaMemcpyHostToDevice,
                                  ctx->stream));
    pd.states = reinterpret_cast<const uint64_t*>(tr + off_st);
  }
  if (int rc = frw_microwalk_batch_dev(ctx, &pd, &d)) return rc;
  if (host->hist)
    FRW_CUDA(ctx, cudaMemcpyAsync(host->hist, ctx->d_hist, bins * 8, cudaMemcpyDeviceToHost,
                                  ctx->stream));
  uint64_t mom[4];
  FRW_CUDA(ctx, cudaMemcpyAsync(mom, ctx->d_mom, 32, cudaMemcpyDeviceToHost, ctx->stream));
  if (host->panels)
    FRW_CUDA(ctx, cudaMemcpyAsync(host->panels, d.panels, cnt * 4, cudaMemcpyDeviceToHost,
                                  ctx->stream));
  if (host->steps)
    FRW_CUDA(ctx, cudaMemcpyAsync(host->steps, d.steps, cnt * 4, cudaMemcpyDeviceToHost,
                                  ctx->stream));
  if (host->cond)
    FRW_CUDA(ctx, cudaMemcpyAsync(host->cond, d.cond, cnt * 4, cudaMemcpyDeviceToHost,
                                  ctx->stream));
  if (host->exit_nd)
    FRW_CUDA(ctx, cudaMemcpyAsync(host->exit_nd, d.exit_nd, cnt * 8, cudaMemcpyDeviceToHost,
                                  ctx->stream));
  FRW_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (host->step_sum) *host->step_sum = mom[0];
  if (host->step_sumsq) *host->step_sumsq = mom[1];
  if (host->cond_exits) *host->cond_exits = mom[2];
  return frw_microwalk_check(ctx);
}

}  // extern "C"
