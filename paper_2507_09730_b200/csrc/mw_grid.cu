// mw_grid.cu -- single-cube MicroWalk on sm_100a (configs C1/C2).
//
// Reference semantics: walk_lattice<GridField> (proj/src/microwalk.cpp:
// 77-156) driven by microwalk_transit (microwalk.cpp:188-197), one
// SplitMix64(seed, stream) per transit in parity mode.
//
// B200 design:
//  * The cube is compiled once into a stencil table: every node gets a
//    16-bit id of its distinct "step record" (the six alphas of Eq. 5 are a
//    function of the node's and its neighbours' permittivities, so a
//    C2-sized cube has ~3k distinct records for 69k nodes).  A record holds
//    the five direction thresholds in the integer domain of the 53-bit
//    uniform: x >= X_d  <=>  fl(x*2^-53*sum) >= acc_d, where acc_d are the
//    reference's in-order partial sums (microwalk.cpp:105-121).  Comparing
//    integers against X_d therefore reproduces the reference's f64 scan bit
//    for bit, with no division and no FP64 on the step path.
//  * The node map (2 B/node) and the record table (24 B/record: the high
//    32 bits of each threshold + the exit codes) are staged into shared
//    memory with one cp.async.bulk per chunk (TMA bulk engine, mbarrier
//    completion).  The low 21 threshold bits stay in global memory and are
//    read only on a high-word tie (probability ~5e-10 per step).
//  * Persistent CTAs, one walker per thread, refilled from a global transit
//    counter; lanes step in phase-aligned super-steps of 4 so Philox blocks
//    and exit bookkeeping are warp-uniform (the "compaction/re-binning" of
//    live walkers: a lane whose transit ends is re-armed with the next
//    transit at the next super-step boundary instead of idling).
//  * Histogram (RED.64 to global), exact u64 step moments and optional
//    per-transit records are fused into the exit path.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <unordered_map>
#include <vector>

#include "frw_internal.h"
#include "frw_rng.cuh"

namespace frw {
namespace {

constexpr int kThreads = 1024;
constexpr int kDirAxis[6] = {0, 0, 1, 1, 2, 2};
constexpr int kDirSign[6] = {-1, +1, -1, +1, -1, +1};

// ---------------------------------------------------------------------------
// host: compile the grid into node map + step records

struct Key {
  uint64_t a, b;
  bool operator==(const Key& o) const { return a == o.a && b == o.b; }
};
struct KeyHash {
  size_t operator()(const Key& k) const {
    return static_cast<size_t>(sm64_mix(k.a ^ sm64_mix(k.b)));
  }
};

// smallest x in [0, 2^53] with fl(x * sum) >= acc * 2^53 (2^53 if none)
uint64_t threshold_of(double acc, double sum) {
  const double target = std::ldexp(acc, 53);
  uint64_t lo = 0, hi = 1ull << 53;  // invariant: answer in [lo, hi]
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (static_cast<double>(mid) * sum >= target)
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

struct Compiled {
  std::vector<uint16_t> map;
  std::vector<uint32_t> rec;     // [R][6]
  std::vector<uint32_t> rec_lo;  // [R][5]
};

int compile_grid(frw_ctx* ctx, int n, const double* eps, const int32_t* mask,
                 Compiled& out) {
  const int nodes = n * n * n;
  std::unordered_map<uint64_t, uint32_t> pal_of;
  std::vector<double> pal;
  std::vector<uint32_t> node_pal(nodes);
  for (int v = 0; v < nodes; ++v) {
    const double e = eps[v];
    if (!(e > 0) || !std::isfinite(e))
      return frw_fail(ctx, FRW_EINVAL, "grid permittivities must be finite and > 0");
    uint64_t bits;
    std::memcpy(&bits, &e, 8);
    auto it = pal_of.find(bits);
    if (it == pal_of.end()) {
      if (pal.size() >= 0xFFF0)
        return frw_fail(ctx, FRW_EINVAL, "more than 65520 distinct permittivities");
      it = pal_of.emplace(bits, static_cast<uint32_t>(pal.size())).first;
      pal.push_back(e);
    }
    node_pal[v] = it->second;
  }
  constexpr uint32_t kSurface = 0xFFFF, kCond = 0xFFFE;
  std::unordered_map<Key, uint32_t, KeyHash> rec_of;
  out.map.resize(nodes);
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        const int v = (k * n + j) * n + i;
        const bool self_cond = mask && mask[v] >= 0;
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
        // conductor voxels are never stepped on; give them a benign key
        const uint32_t self = self_cond ? kCond : node_pal[v];
        Key key{(uint64_t(self) << 48) | (uint64_t(code[0]) << 32) |
                    (uint64_t(code[1]) << 16) | code[2],
                (uint64_t(code[3]) << 32) | (uint64_t(code[4]) << 16) | code[5]};
        auto it = rec_of.find(key);
        if (it == rec_of.end()) {
          const uint32_t r = static_cast<uint32_t>(rec_of.size());
          if (r > 0xFFFF)
            return frw_fail(ctx, FRW_EINVAL, "more than 65536 distinct stencil records");
          it = rec_of.emplace(key, r).first;
          // microwalk.cpp:91-109: alphas and their in-order sum
          double acc[6], sum = 0;
          uint32_t flags = 0;
          const double ev = self_cond ? 1.0 : pal[node_pal[v]];
          for (int d = 0; d < 6; ++d) {
            double a = 1.0;
            if (code[d] == kSurface)
              flags |= 1u << (2 * d);
            else if (code[d] == kCond)
              flags |= 2u << (2 * d);
            else {
              const double en = pal[code[d]];
              a = en / (en + ev);
            }
            sum += a;
            acc[d] = sum;
          }
          for (int d = 0; d < 5; ++d) {
            const uint64_t X = threshold_of(acc[d], sum);
            if (X >= (1ull << 53)) {  // never reached: x < 2^53 always
              out.rec.push_back(0xFFFFFFFFu);
              out.rec_lo.push_back(1u << 21);
            } else {
              out.rec.push_back(static_cast<uint32_t>(X >> 21));
              out.rec_lo.push_back(static_cast<uint32_t>(X & 0x1FFFFFu));
            }
          }
          out.rec.push_back(flags);
        }
        out.map[v] = static_cast<uint16_t>(it->second);
      }
  return FRW_OK;
}

// ---------------------------------------------------------------------------
// device

struct DevGrid {
  const uint16_t* map;
  const uint32_t* rec;
  const uint32_t* rec_lo;
  const int32_t* mask;
  int n;
  int nn;
  int start_idx;
  uint32_t start_pk;
  uint32_t map_bytes;  // padded
  uint32_t rec_bytes;  // padded
};

struct DevParams {
  uint64_t seed;
  uint64_t mixed_seed;
  uint64_t stream_begin;
  long long count;
  int step_cap;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Stage [src, src+bytes) into shared memory with the bulk-copy engine.
__device__ void bulk_stage(void* dst, const void* src, uint32_t bytes,
                           uint64_t* bar) {
  if (threadIdx.x == 0) {
    const uint32_t b = smem_u32(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b),
                 "r"(bytes)
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
  const uint32_t b = smem_u32(bar);
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

// count of thresholds d in 0..4 with x >= X_d, x = (xhi << 21) | xlo;
// the low word (global) is consulted only on a high-word tie
template <class LoFn>
__device__ __forceinline__ int step_dir(uint32_t xhi, const uint32_t* r,
                                        const uint32_t* rec_lo_row,
                                        LoFn&& get_lo) {
  const uint32_t t0 = r[0], t1 = r[1], t2 = r[2], t3 = r[3], t4 = r[4];
  int dir = (xhi > t0) + (xhi > t1) + (xhi > t2) + (xhi > t3) + (xhi > t4);
  const bool tie = (xhi == t0) | (xhi == t1) | (xhi == t2) | (xhi == t3) |
                   (xhi == t4);
  if (__builtin_expect(tie, 0)) {
    const uint32_t xlo = get_lo();
    const uint32_t th[5] = {t0, t1, t2, t3, t4};
    dir = 0;
#pragma unroll
    for (int d = 0; d < 5; ++d)
      dir += (xhi > th[d]) || (xhi == th[d] && xlo >= __ldg(rec_lo_row + d));
  }
  return dir;
}

template <int RNG, bool SMEM>
__global__ void __launch_bounds__(kThreads, 1)
    mw_grid_kernel(DevGrid g, DevParams p, unsigned long long* ctr, int* err,
                   int32_t* out_panel, int32_t* out_steps, int32_t* out_cond,
                   unsigned long long* hist, unsigned long long* m_sum,
                   unsigned long long* m_sq, unsigned long long* m_cx) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ int2 stride[6];  // {node index stride, packed-coordinate stride}

  const uint16_t* map = g.map;
  const uint32_t* rec = g.rec;
  if (SMEM) {
    bulk_stage(smem, g.map, g.map_bytes + g.rec_bytes, &bar);
    map = reinterpret_cast<const uint16_t*>(smem);
    rec = reinterpret_cast<const uint32_t*>(smem + g.map_bytes);
  }
  if (threadIdx.x < 6) {
    const int d = threadIdx.x, ax = d >> 1, s = (d & 1) ? 1 : -1;
    stride[d] = make_int2(s * (ax == 0 ? 1 : ax == 1 ? g.n : g.nn),
                          s * (1 << (10 * ax)));
  }
  __syncthreads();

  const int n = g.n;
  const int cap = p.step_cap;
  unsigned long long ssum = 0, ssq = 0, cexit = 0;

  long long t = static_cast<long long>(atomicAdd(ctr, 1ull));
  long long t_next = static_cast<long long>(atomicAdd(ctr, 1ull));
  bool live = t < p.count;
  int idx = g.start_idx;
  uint32_t pk = g.start_pk;
  int steps = 0;
  uint64_t sm = 0;     // parity: SplitMix64 state
  uint32_t blk = 0;    // philox: 4-step block index within the transit
  if (RNG == FRW_RNG_SPLITMIX_PARITY && live)
    sm = sm64_stream_from_mixed(p.mixed_seed, p.stream_begin + t);

  const uint32_t k0 = static_cast<uint32_t>(p.seed);
  const uint32_t k1 = static_cast<uint32_t>(p.seed >> 32);

  while (__any_sync(0xFFFFFFFFu, live)) {
    // ---- one phase-aligned super-step of 4 lattice steps ----------------
    uint32_t w[4];
    if (RNG == FRW_RNG_PHILOX) {
      const uint64_t id = static_cast<uint64_t>(p.stream_begin + t);
      const U32x4 o = philox4x32_10(
          {static_cast<uint32_t>(id), static_cast<uint32_t>(id >> 32), blk, 0u},
          k0, k1);
      w[0] = o.x; w[1] = o.y; w[2] = o.z; w[3] = o.w;
    }
    int code = 0, xdir = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (live && code == 0 && steps < cap) {
        ++steps;
        uint32_t xhi;
        uint64_t z = 0;
        if (RNG == FRW_RNG_SPLITMIX_PARITY) {
          z = sm64_next(sm);
          xhi = static_cast<uint32_t>(z >> 32);
        } else {
          xhi = w[u];
        }
        const uint32_t r = map[idx];
        const uint32_t* rr = rec + 6 * r;
        const int dir = step_dir(xhi, rr, g.rec_lo + 5 * r, [&]() -> uint32_t {
          if (RNG == FRW_RNG_SPLITMIX_PARITY)
            return static_cast<uint32_t>(z >> 11) & 0x1FFFFFu;
          const uint64_t id = static_cast<uint64_t>(p.stream_begin + t);
          return philox4x32_10({static_cast<uint32_t>(id),
                                static_cast<uint32_t>(id >> 32),
                                static_cast<uint32_t>(steps), 1u},
                               k0, k1).x >> 11;
        });
        const int c = (rr[5] >> (2 * dir)) & 3;
        if (c) {
          code = c;
          xdir = dir;
        } else {
          const int2 s = stride[dir];
          idx += s.x;
          pk += s.y;
        }
      }
    }
    ++blk;
    // ---- exit bookkeeping, batched once per super-step -------------------
    if (live && (code != 0 || steps >= cap)) {
      int32_t panel = -1, cid = -1;
      if (code == 1) {
        const int i = pk & 1023, j = (pk >> 10) & 1023, k = pk >> 20;
        const int ax = xdir >> 1;
        const int uu = ax == 0 ? j : i;
        const int vv = ax == 2 ? j : k;
        panel = (xdir * n + vv) * n + uu;  // sgf.hpp:34-36, sgf.cpp:13-30
        atomicAdd(hist + panel, 1ull);
      } else if (code == 2) {
        cid = g.mask[idx + stride[xdir].x];
        ++cexit;
      } else {
        atomicExch(err, FRW_ESTEPCAP);  // microwalk.cpp:153-155
      }
      if (out_panel) out_panel[t] = panel;
      if (out_steps) out_steps[t] = steps;
      if (out_cond) out_cond[t] = cid;
      ssum += steps;
      ssq += static_cast<unsigned long long>(steps) * steps;
      // re-arm with the prefetched transit, prefetch the following one
      t = t_next;
      live = t < p.count;
      if (live) {
        t_next = static_cast<long long>(atomicAdd(ctr, 1ull));
        idx = g.start_idx;
        pk = g.start_pk;
        steps = 0;
        blk = 0;
        if (RNG == FRW_RNG_SPLITMIX_PARITY)
          sm = sm64_stream_from_mixed(p.mixed_seed, p.stream_begin + t);
      }
    }
  }
  // exact moments: warp reduce then one atomic per warp
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
int launch(frw_ctx* ctx, const frw_mw_params* p, const frw_mw_out* o) {
  const GridTable& G = ctx->grid;
  DevGrid g{G.d_map, G.d_rec, G.d_rec_lo, G.d_mask, G.n, G.n * G.n, G.start_idx,
            0, static_cast<uint32_t>(G.map_bytes), static_cast<uint32_t>(G.rec_bytes)};
  const int c = (G.n - 1) / 2;
  g.start_pk = static_cast<uint32_t>(c | (c << 10) | (c << 20));
  DevParams dp{p->seed, sm64_mix(p->seed), p->stream_begin, p->count,
               p->step_cap > 0 ? p->step_cap : 1000 * G.n * G.n};
  const size_t smem = SMEM ? G.map_bytes + G.rec_bytes : 0;
  auto kern = mw_grid_kernel<RNG, SMEM>;
  if (SMEM)
    FRW_CUDA(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem)));
  FRW_CUDA(ctx, cudaMemsetAsync(ctx->d_ctr, 0, sizeof(unsigned long long), ctx->stream));
  const int blocks = p->blocks > 0 ? p->blocks : ctx->sm_count;
  kern<<<blocks, kThreads, smem, ctx->stream>>>(
      g, dp, ctx->d_ctr, ctx->d_err, o->panels, o->steps, o->cond,
      reinterpret_cast<unsigned long long*>(o->hist),
      reinterpret_cast<unsigned long long*>(o->step_sum ? o->step_sum : ctx->d_mom),
      reinterpret_cast<unsigned long long*>(o->step_sumsq ? o->step_sumsq : ctx->d_mom + 1),
      reinterpret_cast<unsigned long long*>(o->cond_exits ? o->cond_exits : ctx->d_mom + 2));
  FRW_CUDA(ctx, cudaGetLastError());
  return FRW_OK;
}

}  // namespace
}  // namespace frw

using namespace frw;

extern "C" {

int frw_upload_grid(frw_ctx* ctx, int n, const double* eps, const int32_t* mask,
                    double cx, double cy, double cz, double half_width) {
  if (!ctx) return FRW_EINVAL;
  if (n < 1 || n > 1000 || !eps)
    return frw_fail(ctx, FRW_EINVAL, "upload_grid: need 1 <= n <= 1000 and eps");
  if (!(half_width > 0)) return frw_fail(ctx, FRW_EINVAL, "upload_grid: half_width <= 0");
  Compiled cg;
  if (int rc = compile_grid(ctx, n, eps, mask, cg)) return rc;
  FRW_CUDA(ctx, cudaSetDevice(ctx->device));
  GridTable& G = ctx->grid;
  cudaFree(G.d_map);  // also releases d_rec (same allocation)
  cudaFree(G.d_rec_lo);
  cudaFree(G.d_mask);
  G = GridTable{};
  G.n = n;
  G.records = static_cast<int>(cg.rec.size() / 6);
  const int c = (n - 1) / 2;  // start_node, sgf.hpp:58-61
  G.start_idx = (c * n + c) * n + c;
  G.start_is_conductor = mask && mask[G.start_idx] >= 0;
  G.center[0] = cx;
  G.center[1] = cy;
  G.center[2] = cz;
  G.half_width = half_width;
  G.map_bytes = (cg.map.size() * 2 + 15) / 16 * 16;
  G.rec_bytes = (cg.rec.size() * 4 + 15) / 16 * 16;
  // one allocation: map then records, so one bulk stage covers both
  char* blob = nullptr;
  FRW_CUDA(ctx, cudaMalloc(&blob, G.map_bytes + G.rec_bytes));
  G.d_map = reinterpret_cast<uint16_t*>(blob);
  G.d_rec = reinterpret_cast<uint32_t*>(blob + G.map_bytes);
  FRW_CUDA(ctx, cudaMemcpyAsync(G.d_map, cg.map.data(), cg.map.size() * 2,
                                cudaMemcpyHostToDevice, ctx->stream));
  FRW_CUDA(ctx, cudaMemcpyAsync(G.d_rec, cg.rec.data(), cg.rec.size() * 4,
                                cudaMemcpyHostToDevice, ctx->stream));
  FRW_CUDA(ctx, cudaMalloc(&G.d_rec_lo, cg.rec_lo.size() * 4));
  FRW_CUDA(ctx, cudaMemcpyAsync(G.d_rec_lo, cg.rec_lo.data(), cg.rec_lo.size() * 4,
                                cudaMemcpyHostToDevice, ctx->stream));
  if (mask) {
    const size_t nodes = static_cast<size_t>(n) * n * n;
    FRW_CUDA(ctx, cudaMalloc(&G.d_mask, nodes * 4));
    FRW_CUDA(ctx, cudaMemcpyAsync(G.d_mask, mask, nodes * 4, cudaMemcpyHostToDevice,
                                  ctx->stream));
  }
  FRW_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  // the d_map blob is freed through d_map (cudaFree on the base pointer)
  return FRW_OK;
}

int frw_grid_compile(int n, const double* eps, const int32_t* mask, uint16_t* map,
                     uint32_t* rec, uint32_t* rec_lo, int* records) {
  if (n < 1 || n > 1000 || !eps || !records) return FRW_EINVAL;
  frw_ctx tmp;
  Compiled cg;
  if (int rc = compile_grid(&tmp, n, eps, mask, cg)) return rc;
  *records = static_cast<int>(cg.rec.size() / 6);
  if (map) std::memcpy(map, cg.map.data(), cg.map.size() * 2);
  if (rec) std::memcpy(rec, cg.rec.data(), cg.rec.size() * 4);
  if (rec_lo) std::memcpy(rec_lo, cg.rec_lo.data(), cg.rec_lo.size() * 4);
  return FRW_OK;
}

int frw_grid_info(const frw_ctx* ctx, int* records, int* smem_bytes, int* smem_resident) {
  if (!ctx) return FRW_EINVAL;
  const GridTable& G = ctx->grid;
  const size_t bytes = G.map_bytes + G.rec_bytes;
  if (records) *records = G.records;
  if (smem_bytes) *smem_bytes = static_cast<int>(bytes);
  if (smem_resident)
    *smem_resident = bytes + 1024 <= static_cast<size_t>(ctx->max_smem_optin);
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
  if (p->rng_mode != FRW_RNG_SPLITMIX_PARITY && p->rng_mode != FRW_RNG_PHILOX)
    return frw_fail(ctx, FRW_EINVAL, "microwalk_batch: unknown rng mode");
  FRW_CUDA(ctx, cudaSetDevice(ctx->device));
  if (p->count == 0) return FRW_OK;
  const bool smem = G.map_bytes + G.rec_bytes + 1024 <= static_cast<size_t>(ctx->max_smem_optin);
  if (p->rng_mode == FRW_RNG_SPLITMIX_PARITY)
    return smem ? launch<FRW_RNG_SPLITMIX_PARITY, true>(ctx, p, o)
                : launch<FRW_RNG_SPLITMIX_PARITY, false>(ctx, p, o);
  return smem ? launch<FRW_RNG_PHILOX, true>(ctx, p, o)
              : launch<FRW_RNG_PHILOX, false>(ctx, p, o);
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
  const bool per = host->panels || host->steps || host->cond;
  if (per && ctx->tr_cap < static_cast<size_t>(p->count)) {
    cudaFree(ctx->d_tr);
    FRW_CUDA(ctx, cudaMalloc(&ctx->d_tr, static_cast<size_t>(p->count) * 12));
    ctx->tr_cap = p->count;
  }
  FRW_CUDA(ctx, cudaMemsetAsync(ctx->d_hist, 0, bins * 8, ctx->stream));
  FRW_CUDA(ctx, cudaMemsetAsync(ctx->d_mom, 0, 32, ctx->stream));
  FRW_CUDA(ctx, cudaMemsetAsync(ctx->d_err, 0, sizeof(int), ctx->stream));
  frw_mw_out d{};
  d.hist = ctx->d_hist;
  d.step_sum = ctx->d_mom;
  d.step_sumsq = ctx->d_mom + 1;
  d.cond_exits = ctx->d_mom + 2;
  if (host->panels) d.panels = ctx->d_tr;
  if (host->steps) d.steps = ctx->d_tr + p->count;
  if (host->cond) d.cond = ctx->d_tr + 2 * p->count;
  if (int rc = frw_microwalk_batch_dev(ctx, p, &d)) return rc;
  if (host->hist)
    FRW_CUDA(ctx, cudaMemcpyAsync(host->hist, ctx->d_hist, bins * 8, cudaMemcpyDeviceToHost,
                                  ctx->stream));
  uint64_t mom[4];
  FRW_CUDA(ctx, cudaMemcpyAsync(mom, ctx->d_mom, 32, cudaMemcpyDeviceToHost, ctx->stream));
  const size_t cnt = static_cast<size_t>(p->count);
  if (host->panels)
    FRW_CUDA(ctx, cudaMemcpyAsync(host->panels, d.panels, cnt * 4, cudaMemcpyDeviceToHost,
                                  ctx->stream));
  if (host->steps)
    FRW_CUDA(ctx, cudaMemcpyAsync(host->steps, d.steps, cnt * 4, cudaMemcpyDeviceToHost,
                                  ctx->stream));
  if (host->cond)
    FRW_CUDA(ctx, cudaMemcpyAsync(host->cond, d.cond, cnt * 4, cudaMemcpyDeviceToHost,
                                  ctx->stream));
  FRW_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (host->step_sum) *host->step_sum = mom[0];
  if (host->step_sumsq) *host->step_sumsq = mom[1];
  if (host->cond_exits) *host->cond_exits = mom[2];
  return frw_microwalk_check(ctx);
}

}  // extern "C"
