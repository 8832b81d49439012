// fv_oracle.cu -- the reference's full-domain finite-volume capacitance
// solver (proj/src/oracle.cpp:92-213, `reference_capacitance`) on the device.
//
// R^3 voxels over the world box, centres lo + (i + 0.5) h; a voxel inside a
// conductor (conductor_at(p, 0), first declared wins) is that terminal,
// otherwise a free row with the last-declared dielectric's permittivity.
// Face conductances (area/spacing prefactor fpre): free-free
// fpre * 2 e_v e_n / (e_v + e_n); free-wall and free-conductor 2 fpre e_v
// (half spacing).  One Jacobi-preconditioned CG per terminal excitation
// (x0 = 0, |r| <= 1e-9 |b|, at most 200 R iterations, as Eigen's
// ConjugateGradient with its diagonal preconditioner), then
// Q_i = sum over (conductor i | free v) faces of g (V_i - phi_v).
//
// Validation machinery: the end-to-end acceptance
// pin compares walk capacitances against it (acceptance_main.cpp:380-413).
// The CG runs as one cooperative persistent kernel per excitation: grid-wide
// syncs between the SpMV, the updates and the direction update, and
// deterministic reductions (every CTA sums the per-CTA partials in the same
// order).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "frw_internal.h"

namespace cg = cooperative_groups;

namespace frw {
namespace {

constexpr int kFvThreads = 256;

struct FvGrid {
  int R;
  double lo[3], h[3], fpre[3];
};

__global__ void k_fv_classify(FvGrid G, int nc, const double* cbox, int nd, const double* dbox,
                              const double* deps, double bg, double* veps, int* vterm) {
  const long long nv = static_cast<long long>(G.R) * G.R * G.R;
  for (long long v = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; v < nv;
       v += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(v % G.R), j = static_cast<int>((v / G.R) % G.R),
              k = static_cast<int>(v / (static_cast<long long>(G.R) * G.R));
    // oracle.cpp:121-122 voxel centre
    const double p[3] = {G.lo[0] + (i + 0.5) * G.h[0], G.lo[1] + (j + 0.5) * G.h[1],
                         G.lo[2] + (k + 0.5) * G.h[2]};
    double e = bg;  // permittivity_at: last declared dielectric containing p
    for (int d = 0; d < nd; ++d) {
      const double* b = dbox + 6 * d;
      if (p[0] >= b[0] && p[0] <= b[3] && p[1] >= b[1] && p[1] <= b[4] && p[2] >= b[2] &&
          p[2] <= b[5])
        e = deps[d];
    }
    int t = -1;  // conductor_at(p, 0): first declared conductor containing p
    for (int c = 0; c < nc && t < 0; ++c) {
      const double* b = cbox + 6 * c;
      if (p[0] >= b[0] && p[0] <= b[3] && p[1] >= b[1] && p[1] <= b[4] && p[2] >= b[2] &&
          p[2] <= b[5])
        t = c;
    }
    veps[v] = e;
    vterm[v] = t;
  }
}

// the six face conductances of free voxel v; neighbour index or -1 (wall),
// conductor terminal of the neighbour (or -1)
struct Faces {
  double g[6];
  long long nb[6];
  int term[6];
  double diag;
};

__device__ __forceinline__ Faces faces_of(const FvGrid& G, const double* veps, const int* vterm,
                                          long long v) {
  const int R = G.R;
  const long long RR = static_cast<long long>(R) * R;
  const int c[3] = {static_cast<int>(v % R), static_cast<int>((v / R) % R),
                    static_cast<int>(v / RR)};
  const double ev = veps[v];
  Faces f;
  double diag = 0;
#pragma unroll
  for (int dir = 0; dir < 6; ++dir) {
    const int axis = dir >> 1;
    const int nc = c[axis] + ((dir & 1) ? 1 : -1);
    f.term[dir] = -1;
    f.nb[dir] = -1;
    if (nc < 0 || nc >= R) {  // grounded world wall, half spacing
      f.g[dir] = 2.0 * G.fpre[axis] * ev;
      diag += f.g[dir];
      continue;
    }
    const long long st = axis == 0 ? 1 : (axis == 1 ? R : RR);
    const long long u = (dir & 1) ? v + st : v - st;
    const int tu = vterm[u];
    if (tu >= 0) {  // conductor surface on the shared face, half spacing
      f.g[dir] = 2.0 * G.fpre[axis] * ev;
      f.term[dir] = tu;
      diag += f.g[dir];
      continue;
    }
    const double en = veps[u];
    f.g[dir] = G.fpre[axis] * 2.0 * ev * en / (ev + en);  // oracle.cpp:171
    f.nb[dir] = u;
    diag += f.g[dir];
  }
  f.diag = diag;
  return f;
}

__device__ __forceinline__ double grid_sum(const double* partial, int nblocks, double* red) {
  // every CTA sums the per-CTA partials in the same order (deterministic)
  double s = 0;
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x) s += partial[b];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = s;
  __syncthreads();
  double t = 0;
  if (threadIdx.x == 0) {
    for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) t += red[q];
    red[32] = t;
  }
  __syncthreads();
  const double r = red[32];
  __syncthreads();
  return r;
}

__device__ __forceinline__ void block_partial(double v, double* red, double* out) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) t += red[q];
    *out = t;
  }
  __syncthreads();
}

struct CgBufs {
  double *x, *r, *p, *t, *dinv;
  double *part_a, *part_b, *part_c;  // [gridDim] per-CTA partials
  int* iters;
  double* relres;
};

__global__ void __launch_bounds__(kFvThreads)
    k_fv_cg(FvGrid G, const double* veps, const int* vterm, int term, CgBufs B, long maxit,
            double tol) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[40];
  const long long nv = static_cast<long long>(G.R) * G.R * G.R;
  const long long gstride = static_cast<long long>(gridDim.x) * blockDim.x;
  const long long g0 = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  // b = Dirichlet couplings to the excited terminal (oracle.cpp:194-196)
  double bb = 0, rz = 0;
  for (long long v = g0; v < nv; v += gstride) {
    double b = 0, di = 0;
    if (vterm[v] < 0) {
      const Faces f = faces_of(G, veps, vterm, v);
#pragma unroll
      for (int d = 0; d < 6; ++d)
        if (f.term[d] == term) b += f.g[d];
      di = 1.0 / f.diag;
    }
    B.dinv[v] = di;
    B.x[v] = 0.0;
    B.r[v] = b;
    B.p[v] = b * di;
    bb += b * b;
    rz += b * (b * di);
  }
  block_partial(bb, red, B.part_a + blockIdx.x);
  block_partial(rz, red, B.part_b + blockIdx.x);
  grid.sync();
  const double b2 = grid_sum(B.part_a, gridDim.x, red);
  rz = grid_sum(B.part_b, gridDim.x, red);
  grid.sync();
  const double thresh = tol * tol * b2;
  double res2 = b2;
  long it = 0;
  if (b2 == 0.0) res2 = 0.0;  // no coupling: phi = 0
  while (res2 > thresh && it < maxit) {
    double pt = 0;
    for (long long v = g0; v < nv; v += gstride) {
      double acc = 0;
      if (vterm[v] < 0) {
        const Faces f = faces_of(G, veps, vterm, v);
        acc = f.diag * B.p[v];
#pragma unroll
        for (int d = 0; d < 6; ++d)
          if (f.nb[d] >= 0) acc -= f.g[d] * B.p[f.nb[d]];
      }
      B.t[v] = acc;
      pt += B.p[v] * acc;
    }
    block_partial(pt, red, B.part_a + blockIdx.x);
    grid.sync();
    const double alpha = rz / grid_sum(B.part_a, gridDim.x, red);
    double rr = 0, rzn = 0;
    for (long long v = g0; v < nv; v += gstride) {
      B.x[v] += alpha * B.p[v];
      const double rv = B.r[v] - alpha * B.t[v];
      B.r[v] = rv;
      rr += rv * rv;
      rzn += rv * (rv * B.dinv[v]);
    }
    block_partial(rr, red, B.part_b + blockIdx.x);
    block_partial(rzn, red, B.part_c + blockIdx.x);
    grid.sync();
    res2 = grid_sum(B.part_b, gridDim.x, red);
    const double rz_new = grid_sum(B.part_c, gridDim.x, red);
    ++it;
    if (res2 <= thresh) break;
    const double beta = rz_new / rz;
    rz = rz_new;
    for (long long v = g0; v < nv; v += gstride) B.p[v] = B.r[v] * B.dinv[v] + beta * B.p[v];
    grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *B.iters = static_cast<int>(it);
    *B.relres = b2 > 0 ? sqrt(res2 / b2) : 0.0;
  }
}

// Q_i += g (V_i - phi_v) over (conductor i | free v) faces (oracle.cpp:204-209)
__global__ void k_fv_charge(FvGrid G, const double* veps, const int* vterm, int term,
                            const double* phi, double* q) {
  const long long nv = static_cast<long long>(G.R) * G.R * G.R;
  for (long long v = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; v < nv;
       v += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (vterm[v] >= 0) continue;
    const Faces f = faces_of(G, veps, vterm, v);
#pragma unroll
    for (int d = 0; d < 6; ++d)
      if (f.term[d] >= 0)
        atomicAdd(q + f.term[d], f.g[d] * ((f.term[d] == term ? 1.0 : 0.0) - phi[v]));
  }
}

}  // namespace
}  // namespace frw

using namespace frw;

extern "C" int frw_reference_capacitance(frw_ctx* ctx, const frw_structure* s, int resolution,
                                         double* cap, double* residual) {
  if (!ctx || !s || !cap) return FRW_EINVAL;
  if (resolution < 16)
    return frw_fail(ctx, FRW_EINVAL, "reference_capacitance: resolution < 16");
  const long long R = resolution, nv = R * R * R;
  if (nv > 3500000)
    return frw_fail(ctx, FRW_EINVAL, "reference_capacitance: resolution too large, lower it");
  if (s->n_cond < 1) return frw_fail(ctx, FRW_EINVAL, "reference_capacitance: no conductors");
  FRW_CUDA(ctx, cudaSetDevice(ctx->device));
  FvGrid G;
  G.R = resolution;
  for (int a = 0; a < 3; ++a) {
    G.lo[a] = s->world[a];
    G.h[a] = (s->world[3 + a] - s->world[a]) / R;  // ext / R
  }
  G.fpre[0] = G.h[1] * G.h[2] / G.h[0];
  G.fpre[1] = G.h[0] * G.h[2] / G.h[1];
  G.fpre[2] = G.h[0] * G.h[1] / G.h[2];
  const int T = s->n_cond;
  std::vector<double*> dbl;
  auto alloc = [&](size_t n) {
    double* p = nullptr;
    if (cudaMalloc(&p, 8 * std::max<size_t>(n, 1)) != cudaSuccess) return static_cast<double*>(nullptr);
    dbl.push_back(p);
    return p;
  };
  int* vterm = nullptr;
  int* iters = nullptr;
  double* veps = alloc(nv);
  double* cb = alloc(6 * size_t(T));
  double* db = alloc(6 * size_t(std::max(s->n_diel, 1)));
  double* de = alloc(std::max(s->n_diel, 1));
  CgBufs B{};
  B.x = alloc(nv);
  B.r = alloc(nv);
  B.p = alloc(nv);
  B.t = alloc(nv);
  B.dinv = alloc(nv);
  double* q = alloc(T);
  double* rel = alloc(1);
  int blocks_per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_fv_cg, kFvThreads, 0);
  const int grid = std::max(1, blocks_per_sm) * ctx->sm_count;
  B.part_a = alloc(grid);
  B.part_b = alloc(grid);
  B.part_c = alloc(grid);
  B.relres = rel;
  bool ok = cudaMalloc(&vterm, 4 * nv) == cudaSuccess && cudaMalloc(&iters, 4) == cudaSuccess;
  for (double* p : dbl) ok = ok && p;
  int status = FRW_OK;
  auto cleanup = [&] {
    for (double* p : dbl) cudaFree(p);
    cudaFree(vterm);
    cudaFree(iters);
  };
  if (!ok) {
    cleanup();
    return frw_fail(ctx, FRW_ENOMEM, "reference_capacitance: device allocation failed");
  }
  B.iters = iters;
  cudaStream_t st = ctx->stream;
  cudaMemcpyAsync(cb, s->cond_box, 48 * size_t(T), cudaMemcpyHostToDevice, st);
  if (s->n_diel > 0) {
    cudaMemcpyAsync(db, s->diel_box, 48 * size_t(s->n_diel), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(de, s->diel_eps, 8 * size_t(s->n_diel), cudaMemcpyHostToDevice, st);
  }
  k_fv_classify<<<ctx->sm_count * 8, 256, 0, st>>>(G, T, cb, s->n_diel, db, de, s->background_eps,
                                                    veps, vterm);
  double worst = 0;
  const long maxit = 200L * resolution;  // oracle.cpp:188
  const double tol = 1e-9;               // oracle.cpp:187
  std::vector<double> qh(T);
  for (int t = 0; t < T && status == FRW_OK; ++t) {
    int term = t;
    long mi = maxit;
    double tl = tol;
    const double* cveps = veps;
    const int* cvterm = vterm;
    void* args[] = {&G, &cveps, &cvterm, &term, &B, &mi, &tl};
    if (cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_fv_cg), grid, kFvThreads, args, 0,
                                    st) != cudaSuccess) {
      status = frw_fail(ctx, FRW_ECUDA, "reference_capacitance: cooperative launch failed");
      break;
    }
    cudaMemsetAsync(q, 0, 8 * size_t(T), st);
    k_fv_charge<<<ctx->sm_count * 8, 256, 0, st>>>(G, veps, vterm, t, B.x, q);
    int it = 0;
    double rr = 0;
    cudaMemcpyAsync(qh.data(), q, 8 * size_t(T), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&it, iters, 4, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&rr, rel, 8, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) {
      status = frw_fail(ctx, FRW_ECUDA, "reference_capacitance: solve failed");
      break;
    }
    if (it >= maxit && rr > tol) {
      status = frw_fail(ctx, FRW_ESOLVE,
                        "reference_capacitance: solver failed to converge, lower the resolution");
      break;
    }
    worst = std::max(worst, rr);
    for (int i = 0; i < T; ++i) cap[static_cast<size_t>(i) * T + t] = qh[i] * (8.8541878128e-12 * 1e-9);
  }
  if (residual) *residual = worst;
  cleanup();
  return status;
}
