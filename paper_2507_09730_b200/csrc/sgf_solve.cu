// sgf_solve.cu -- stratified-SGF miss solver on the device.
//
// Solves the canonical unit-pitch grid of a ProfileKey (sgf_cache.cpp:78-96:
// eps(i,j,k) = layers[{i,j,k}[axis]], half width n/2) for the surface
// Green's function and its three gradient kernels, restating
// proj/src/sgf.cpp:57-290:
//   s_ii = diag(eps) A_II, bit-symmetric entries -(e_v e_i)/(e_v + e_i),
//   diagonal e_v * sum(alpha) with alpha = e_i/(e_i+e_v) (1 on the faces);
//   adjoint trick: s_ii z = b, probs = A_IB^T (eps .* z);
//   b = e_c (probs) and e_{c+a} - e_{c-a} (kernel a, central difference,
//   one-sided at a lattice face), divided by the pitch span;
//   Jacobi-PCG from zero, stop at |r|^2 < (1e-10)^2 |b|^2, cap 20*rows.
// One CTA per (key, right-hand side); the stencil of a stratified grid is a
// function of the layer index along the key axis only, so the per-layer
// coefficients live in shared memory and the SpMV is division free.  The
// four Krylov vectors of a CTA stay L2-resident in a scratch slab.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "frw_internal.h"

namespace frw {
namespace {

constexpr int kSolveThreads = 1024;
constexpr int kMaxN = 64;

struct Layer {
  double e;       // permittivity
  double a_dn;    // alpha towards layer t-1: e_{t-1}/(e_{t-1}+e_t)
  double a_up;    // alpha towards layer t+1
  double s_dn;    // s_ii entry towards t-1: -(e_t e_{t-1})/(e_t + e_{t-1})
  double s_up;
  double s_perp;  // within the layer: -(e e)/(e + e)
};

__device__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < (blockDim.x >> 5) ? red[l] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if (l == 0) red[32] = v;
  }
  __syncthreads();
  return red[32];
}

struct Row {
  double diag;
  double off[6];  // 0 where the face absorbs
};

// row v of s_ii (sgf.cpp:99-137, same summation order for the row sum)
__device__ __forceinline__ Row make_row(const Layer* L, int n, int axis, int i, int j, int k) {
  const int c[3] = {i, j, k};
  const int t = c[axis];
  Row r;
  double rs = 0;
#pragma unroll
  for (int d = 0; d < 6; ++d) {
    const int a = d >> 1;
    const int nb = c[a] + ((d & 1) ? 1 : -1);
    if (nb < 0 || nb >= n) {
      rs += 1.0;
      r.off[d] = 0.0;
      continue;
    }
    if (a == axis) {
      rs += (d & 1) ? L[t].a_up : L[t].a_dn;
      r.off[d] = (d & 1) ? L[t].s_up : L[t].s_dn;
    } else {
      rs += 0.5;  // e/(e+e)
      r.off[d] = L[t].s_perp;
    }
  }
  r.diag = L[t].e * rs;
  return r;
}

__global__ void __launch_bounds__(kSolveThreads)
    k_sgf_pcg(int n, const int* axes, const double* layers, double* slab, double* out,
              int* status) {
  __shared__ Layer L[kMaxN];
  __shared__ double red[33];
  const int job = blockIdx.x;
  const int key = job >> 2, rhs = job & 3;
  const int axis = axes[key];
  const double* lay = layers + static_cast<size_t>(key) * n;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const double e = lay[t];
    Layer x;
    x.e = e;
    x.s_perp = -(e * e) / (e + e);
    x.a_dn = x.s_dn = x.a_up = x.s_up = 0;
    if (t > 0) {
      const double ei = lay[t - 1];
      x.a_dn = ei / (ei + e);
      x.s_dn = -(e * ei) / (e + ei);
    }
    if (t + 1 < n) {
      const double ei = lay[t + 1];
      x.a_up = ei / (ei + e);
      x.s_up = -(e * ei) / (e + ei);
    }
    L[t] = x;
  }
  __syncthreads();
  const int m = n * n * n, nn = n * n;
  const int P = 6 * nn;
  double* x = slab + static_cast<size_t>(job) * 4 * m;
  double* r = x + m;
  double* p = r + m;
  double* t = p + m;
  double* o = out + static_cast<size_t>(job) * P;
  const int c = (n - 1) / 2;
  const int crow = (c * n + c) * n + c;
  // right-hand side (sgf.cpp:243 and :265-283)
  int plus = -1, minus = -1;
  double denom = 1.0;
  if (rhs == 0) {
    plus = crow;
  } else {
    const int a = rhs - 1;
    const int st = a == 0 ? 1 : a == 1 ? n : nn;
    const bool up = c + 1 < n, dn = c - 1 >= 0;
    if (up && dn) {
      plus = crow + st;
      minus = crow - st;
      denom = 2.0;  // 2 * pitch, unit pitch
    } else if (up) {
      plus = crow + st;
      minus = crow;
    } else if (dn) {
      plus = crow;
      minus = crow - st;
    }
  }
  if (plus < 0) {  // n = 1: zero kernel
    for (int q = threadIdx.x; q < P; q += blockDim.x) o[q] = 0.0;
    return;
  }
  const int stride[6] = {-1, 1, -n, n, -nn, nn};
  double rr_loc = 0, rz_loc = 0;
  for (int v = threadIdx.x; v < m; v += blockDim.x) {
    const double b = (v == plus ? 1.0 : 0.0) - (v == minus ? 1.0 : 0.0);
    x[v] = 0.0;
    r[v] = b;
    const int i = v % n, j = (v / n) % n, k = v / nn;
    const Row R = make_row(L, n, axis, i, j, k);
    p[v] = b / R.diag;
    rr_loc += b * b;
    rz_loc += b * (b / R.diag);
  }
  const double b2 = block_sum(rr_loc, red);
  const double thresh = 1e-20 * b2;
  double rz = block_sum(rz_loc, red);
  double res2 = b2;
  const long cap = 20L * m;
  long it = 0;
  while (res2 >= thresh && it < cap) {
    // t = s_ii p, <p, t>
    double pt = 0;
    for (int v = threadIdx.x; v < m; v += blockDim.x) {
      const int i = v % n, j = (v / n) % n, k = v / nn;
      const Row R = make_row(L, n, axis, i, j, k);
      double acc = R.diag * p[v];
#pragma unroll
      for (int d = 0; d < 6; ++d)
        if (R.off[d] != 0.0) acc += R.off[d] * p[v + stride[d]];
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
      const int i = v % n, j = (v / n) % n, k = v / nn;
      rzn += rv * (rv / make_row(L, n, axis, i, j, k).diag);
    }
    res2 = block_sum(rr, red);
    const double rz_new = block_sum(rzn, red);
    ++it;
    if (res2 < thresh) break;
    const double beta = rz_new / rz;
    rz = rz_new;
    __syncthreads();
    for (int v = threadIdx.x; v < m; v += blockDim.x) {
      const int i = v % n, j = (v / n) % n, k = v / nn;
      p[v] = r[v] / make_row(L, n, axis, i, j, k).diag + beta * p[v];
    }
    __syncthreads();
  }
  if (res2 >= thresh && threadIdx.x == 0) atomicExch(status, FRW_ESOLVE);
  __syncthreads();
  // boundary row A_IB^T (eps .* z), panel = (face*n + v)*n + u (sgf.hpp:34-36)
  for (int q = threadIdx.x; q < P; q += blockDim.x) {
    const int face = q / nn, rem = q - face * nn;
    const int u = rem % n, w = rem / n;
    const int a = face >> 1;
    const int edge = (face & 1) ? n - 1 : 0;
    int ci[3];
    ci[a] = edge;
    ci[a == 0 ? 1 : 0] = u;
    ci[a == 2 ? 1 : 2] = w;
    const int v = (ci[2] * n + ci[1]) * n + ci[0];
    o[q] = L[ci[axis]].e * x[v] / denom;
  }
}

// ---- general (unmasked) grids: solve_sgf / expected_steps of a materialised
// DielectricGrid (sgf.cpp:57-299).  The seven s_ii coefficients of every row
// are precomputed once per job (they hold divisions); the PCG is that of
// k_sgf_pcg.  Right-hand sides: 0 e_c (probs), 1..3 gradient kernels,
// 4 expected steps (s_ii t = eps .* rowsum, sgf.cpp:292-299).
__global__ void k_grid_coeffs(int n, int count, const double* eps, double* coef) {
  const size_t m = static_cast<size_t>(n) * n * n;
  const int nn = n * n;
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; q < m * count;
       q += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t g = q / m;
    const int v = static_cast<int>(q - g * m);
    const double* e = eps + g * m;
    const int c[3] = {v % n, (v / n) % n, v / nn};
    const double ev = e[v];
    double* o = coef + (g * m + v) * 8;
    double rs = 0;
#pragma unroll
    for (int d = 0; d < 6; ++d) {
      const int a = d >> 1;
      const int nb = c[a] + ((d & 1) ? 1 : -1);
      if (nb < 0 || nb >= n) {
        rs += 1.0;
        o[1 + d] = 0.0;
        continue;
      }
      const int st = a == 0 ? 1 : (a == 1 ? n : nn);
      const double ei = e[(d & 1) ? v + st : v - st];
      rs += ei / (ei + ev);
      o[1 + d] = -(ev * ei) / (ev + ei);
    }
    o[0] = ev * rs;  // diagonal
    o[7] = rs;       // row sum of alphas (expected-steps right-hand side)
  }
}

__global__ void __launch_bounds__(kSolveThreads)
    k_grid_pcg(int n, const double* eps, const double* coef, double hw, double* slab,
               double* out, double* steps, int* status) {
  __shared__ double red[33];
  const int job = blockIdx.x;
  const int g = job / 5, rhs = job % 5;
  const int m = n * n * n, nn = n * n;
  const int P = 6 * nn;
  const double* e = eps + static_cast<size_t>(g) * m;
  const double* cf = coef + static_cast<size_t>(g) * m * 8;
  double* x = slab + static_cast<size_t>(job) * 4 * m;
  double* r = x + m;
  double* p = r + m;
  double* t = p + m;
  double* o = out + static_cast<size_t>(job) * P;
  const int c = (n - 1) / 2;
  const int crow = (c * n + c) * n + c;
  const double pitch = 2.0 * hw / n;
  int plus = -1, minus = -1;
  double denom = 1.0;
  if (rhs == 0) {
    plus = crow;
  } else if (rhs <= 3) {
    const int a = rhs - 1;
    const int st = a == 0 ? 1 : a == 1 ? n : nn;
    const bool up = c + 1 < n, dn = c - 1 >= 0;
    if (up && dn) {
      plus = crow + st;
      minus = crow - st;
      denom = 2.0 * pitch;
    } else if (up) {
      plus = crow + st;
      minus = crow;
      denom = pitch;
    } else if (dn) {
      plus = crow;
      minus = crow - st;
      denom = pitch;
    }
    if (plus < 0) {  // n = 1: zero kernel
      for (int q = threadIdx.x; q < P; q += blockDim.x) o[q] = 0.0;
      return;
    }
  }
  const int stride[6] = {-1, 1, -n, n, -nn, nn};
  double rr_loc = 0, rz_loc = 0;
  for (int v = threadIdx.x; v < m; v += blockDim.x) {
    const double* rc = cf + static_cast<size_t>(v) * 8;
    const double b = rhs == 4 ? e[v] * rc[7]
                              : (v == plus ? 1.0 : 0.0) - (v == minus ? 1.0 : 0.0);
    x[v] = 0.0;
    r[v] = b;
    p[v] = b / rc[0];
    rr_loc += b * b;
    rz_loc += b * (b / rc[0]);
  }
  const double b2 = block_sum(rr_loc, red);
  const double thresh = 1e-20 * b2;
  double rz = block_sum(rz_loc, red);
  double res2 = b2;
  const long cap = 20L * m;
  long it = 0;
  while (res2 >= thresh && it < cap) {
    double pt = 0;
    for (int v = threadIdx.x; v < m; v += blockDim.x) {
      const double* rc = cf + static_cast<size_t>(v) * 8;
      double acc = rc[0] * p[v];
#pragma unroll
      for (int d = 0; d < 6; ++d)
        if (rc[1 + d] != 0.0) acc += rc[1 + d] * p[v + stride[d]];
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
      rzn += rv * (rv / cf[static_cast<size_t>(v) * 8]);
    }
    res2 = block_sum(rr, red);
    const double rz_new = block_sum(rzn, red);
    ++it;
    if (res2 < thresh) break;
    const double beta = rz_new / rz;
    rz = rz_new;
    __syncthreads();
    for (int v = threadIdx.x; v < m; v += blockDim.x)
      p[v] = r[v] / cf[static_cast<size_t>(v) * 8] + beta * p[v];
    __syncthreads();
  }
  if (res2 >= thresh && b2 > 0 && threadIdx.x == 0) atomicExch(status, FRW_ESOLVE);
  __syncthreads();
  if (rhs == 4) {
    if (threadIdx.x == 0) steps[g] = x[crow];
    return;
  }
  for (int q = threadIdx.x; q < P; q += blockDim.x) {
    const int face = q / nn, rem = q - face * nn;
    const int u = rem % n, w = rem / n;
    const int a = face >> 1;
    int ci[3];
    ci[a] = (face & 1) ? n - 1 : 0;
    ci[a == 0 ? 1 : 0] = u;
    ci[a == 2 ? 1 : 2] = w;
    const int v = (ci[2] * n + ci[1]) * n + ci[0];
    o[q] = e[v] * x[v] / denom;
  }
}

}  // namespace
}  // namespace frw

using namespace frw;

extern "C" int frw_sgf_solve(frw_ctx* ctx, int n, int count, const int* axes,
                             const double* layers, double* probs, double* kernels) {
  if (!ctx || !axes || !layers || !probs) return FRW_EINVAL;
  if (n < 1 || n > kMaxN || count < 0)
    return frw_fail(ctx, FRW_EINVAL, "sgf_solve: need 1 <= n <= 64");
  if (count == 0) return FRW_OK;
  for (int q = 0; q < count; ++q)
    if (axes[q] < 0 || axes[q] > 2) return frw_fail(ctx, FRW_EINVAL, "sgf_solve: bad axis");
  FRW_CUDA(ctx, cudaSetDevice(ctx->device));
  const size_t m = static_cast<size_t>(n) * n * n, P = 6ull * n * n;
  // bounded scratch: solve in chunks of keys
  const int chunk = std::min(count, 512);
  double *d_lay = nullptr, *slab = nullptr, *out = nullptr;
  int *d_ax = nullptr, *d_st = nullptr;
  FRW_CUDA(ctx, cudaMalloc(&d_lay, 8 * static_cast<size_t>(chunk) * n));
  FRW_CUDA(ctx, cudaMalloc(&d_ax, 4 * static_cast<size_t>(chunk)));
  FRW_CUDA(ctx, cudaMalloc(&slab, 8 * 4 * m * 4 * static_cast<size_t>(chunk)));
  FRW_CUDA(ctx, cudaMalloc(&out, 8 * P * 4 * static_cast<size_t>(chunk)));
  FRW_CUDA(ctx, cudaMalloc(&d_st, 4));
  FRW_CUDA(ctx, cudaMemsetAsync(d_st, 0, 4, ctx->stream));
  std::vector<double> h(P * 4 * static_cast<size_t>(chunk));
  int rc = FRW_OK;
  for (int k0 = 0; k0 < count && rc == FRW_OK; k0 += chunk) {
    const int kc = std::min(chunk, count - k0);
    cudaMemcpyAsync(d_lay, layers + static_cast<size_t>(k0) * n, 8 * static_cast<size_t>(kc) * n,
                    cudaMemcpyHostToDevice, ctx->stream);
    cudaMemcpyAsync(d_ax, axes + k0, 4 * static_cast<size_t>(kc), cudaMemcpyHostToDevice,
                    ctx->stream);
    k_sgf_pcg<<<4 * kc, kSolveThreads, 0, ctx->stream>>>(n, d_ax, d_lay, slab, out, d_st);
    cudaMemcpyAsync(h.data(), out, 8 * P * 4 * static_cast<size_t>(kc), cudaMemcpyDeviceToHost,
                    ctx->stream);
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
      rc = frw_fail(ctx, FRW_ECUDA, "sgf_solve: kernel failed");
      break;
    }
    for (int q = 0; q < kc; ++q) {
      const double* pr = &h[(static_cast<size_t>(q) * 4) * P];
      double sum = 0, lo = 0;
      for (size_t b = 0; b < P; ++b) {
        sum += pr[b];
        lo = std::min(lo, pr[b]);
      }
      if (std::fabs(sum - 1.0) > 1e-9 || lo < -1e-9) {  // sgf.cpp:249-253
        rc = frw_fail(ctx, FRW_ESOLVE, "transition cube solve failed normalization check");
        break;
      }
      double* po = probs + static_cast<size_t>(k0 + q) * P;
      for (size_t b = 0; b < P; ++b) po[b] = std::max(pr[b], 0.0);
      if (kernels)
        std::copy(pr + P, pr + 4 * P, kernels + static_cast<size_t>(k0 + q) * 3 * P);
    }
  }
  int st = 0;
  cudaMemcpy(&st, d_st, 4, cudaMemcpyDeviceToHost);
  if (rc == FRW_OK && st) rc = frw_fail(ctx, FRW_ESOLVE, "transition cube solve failed: PCG did not converge");
  cudaFree(d_lay);
  cudaFree(d_ax);
  cudaFree(slab);
  cudaFree(out);
  cudaFree(d_st);
  return rc;
}

extern "C" int frw_grid_sgf_solve(frw_ctx* ctx, int n, int count, const double* eps,
                                  double half_width, double* probs, double* kernels,
                                  double* steps) {
  if (!ctx || !eps || (!probs && !kernels && !steps)) return FRW_EINVAL;
  if (n < 1 || n > kMaxN || count < 0 || !(half_width > 0))
    return frw_fail(ctx, FRW_EINVAL, "grid_sgf_solve: need 1 <= n <= 64, half_width > 0");
  if (count == 0) return FRW_OK;
  const size_t m = static_cast<size_t>(n) * n * n, P = 6ull * n * n;
  for (size_t q = 0; q < m * count; ++q)
    if (!(eps[q] > 0) || !std::isfinite(eps[q]))
      return frw_fail(ctx, FRW_EINVAL, "grid_sgf_solve: permittivities must be finite and > 0");
  FRW_CUDA(ctx, cudaSetDevice(ctx->device));
  const int chunk = std::min(count, 256);
  double *d_eps = nullptr, *coef = nullptr, *slab = nullptr, *out = nullptr, *d_steps = nullptr;
  int* d_st = nullptr;
  FRW_CUDA(ctx, cudaMalloc(&d_eps, 8 * m * chunk));
  FRW_CUDA(ctx, cudaMalloc(&coef, 64 * m * chunk));
  FRW_CUDA(ctx, cudaMalloc(&slab, 8 * 4 * m * 5 * static_cast<size_t>(chunk)));
  FRW_CUDA(ctx, cudaMalloc(&out, 8 * P * 5 * static_cast<size_t>(chunk)));
  FRW_CUDA(ctx, cudaMalloc(&d_steps, 8 * static_cast<size_t>(chunk)));
  FRW_CUDA(ctx, cudaMalloc(&d_st, 4));
  FRW_CUDA(ctx, cudaMemsetAsync(d_st, 0, 4, ctx->stream));
  std::vector<double> h(P * 5 * static_cast<size_t>(chunk)), hs(chunk);
  int rc = FRW_OK;
  for (int g0 = 0; g0 < count && rc == FRW_OK; g0 += chunk) {
    const int gc = std::min(chunk, count - g0);
    cudaMemcpyAsync(d_eps, eps + m * g0, 8 * m * gc, cudaMemcpyHostToDevice, ctx->stream);
    k_grid_coeffs<<<ctx->sm_count * 4, 256, 0, ctx->stream>>>(n, gc, d_eps, coef);
    k_grid_pcg<<<5 * gc, kSolveThreads, 0, ctx->stream>>>(n, d_eps, coef, half_width, slab, out,
                                                           d_steps, d_st);
    cudaMemcpyAsync(h.data(), out, 8 * P * 5 * static_cast<size_t>(gc), cudaMemcpyDeviceToHost,
                    ctx->stream);
    cudaMemcpyAsync(hs.data(), d_steps, 8 * static_cast<size_t>(gc), cudaMemcpyDeviceToHost,
                    ctx->stream);
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
      rc = frw_fail(ctx, FRW_ECUDA, "grid_sgf_solve: kernel failed");
      break;
    }
    for (int q = 0; q < gc; ++q) {
      const double* pr = &h[static_cast<size_t>(q) * 5 * P];
      double sum = 0, lo = 0;
      for (size_t b = 0; b < P; ++b) {
        sum += pr[b];
        lo = std::min(lo, pr[b]);
      }
      if (std::fabs(sum - 1.0) > 1e-9 || lo < -1e-9) {  // sgf.cpp:249-253
        rc = frw_fail(ctx, FRW_ESOLVE, "transition cube solve failed normalization check");
        break;
      }
      if (probs) {
        double* po = probs + static_cast<size_t>(g0 + q) * P;
        for (size_t b = 0; b < P; ++b) po[b] = std::max(pr[b], 0.0);
      }
      if (kernels) std::copy(pr + P, pr + 4 * P, kernels + static_cast<size_t>(g0 + q) * 3 * P);
      if (steps) steps[g0 + q] = hs[q];
    }
  }
  int st = 0;
  cudaMemcpy(&st, d_st, 4, cudaMemcpyDeviceToHost);
  if (rc == FRW_OK && st)
    rc = frw_fail(ctx, FRW_ESOLVE, "transition cube solve failed: PCG did not converge");
  cudaFree(d_eps);
  cudaFree(coef);
  cudaFree(slab);
  cudaFree(out);
  cudaFree(d_steps);
  cudaFree(d_st);
  return rc;
}
