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
// The stratified system is separable and solved directly (k_sgf_direct);
// general grids use the matrix-free Jacobi-PCG of k_grid_pcg.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "frw_internal.h"

namespace frw {
namespace {

constexpr int kSolveThreads = 1024;
constexpr int kMaxN = 128;     // stratified keys (direct solve): the walk engine's grid_n cap
constexpr int kGridMaxN = 64;  // general grids (Jacobi-PCG, FDM / validate-sgf)

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

// ---- stratified keys: separable direct solve --------------------------------
// On the canonical grid of a stratified key the permittivity depends only on
// the layer index t along the key axis, so
//   s_ii = A (x) I (x) I + E (x) (M (x) I + I (x) M),
// with A the axial tridiagonal operator of the layers (s_ii entries
// -(e_t e_t')/(e_t + e_t'), diagonal e_t (alpha_dn + alpha_up)), E = diag(e_t)
// and M the 1-D operator of a uniform row with the half-spacing absorbing
// faces: tridiag(-1/2, 1, -1/2) with 3/2 at both ends.  2M is the
// cell-centred Dirichlet Laplacian, diagonalised by the DST-II basis
//   q_k[i] = c_k sin(pi k (i + 1/2) / n),  lambda_k = 2 sin^2(pi k / 2n).
// Each of the n^2 perpendicular modes is then one tridiagonal system
// (A + (lambda_k1 + lambda_k2) E) z = beta along the key axis (Thomas), and
// the boundary values are transformed back.  Exact to rounding -- the same
// system the reference solves by Jacobi-PCG to 1e-10 (sgf.cpp:162-290).
constexpr int kDirectThreads = 256;

__device__ __forceinline__ double dst2(int n, int k, int i) {  // q_k[i], k = 1..n
  const double c = k == n ? sqrt(1.0 / n) : sqrt(2.0 / n);
  return c * sin(M_PI * k * (i + 0.5) / n);
}

__global__ void __launch_bounds__(kDirectThreads)
    k_sgf_direct(int n, const int* axes, const double* layers, double* scratch, double* out) {
  __shared__ double e[kMaxN], adiag[kMaxN], aoff[kMaxN], lam[kMaxN];
  extern __shared__ double q[];  // [n * n]: q[k * n + i], k = 0..n-1 for modes 1..n
  const int key = blockIdx.x;
  const int axis = axes[key];
  const int nn = n * n, m = nn * n, P = 6 * nn;
  const double* lay = layers + static_cast<size_t>(key) * n;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const double et = lay[t];
    e[t] = et;
    const double adn = t > 0 ? lay[t - 1] / (lay[t - 1] + et) : 1.0;
    const double aup = t + 1 < n ? lay[t + 1] / (lay[t + 1] + et) : 1.0;
    adiag[t] = et * (adn + aup);
    aoff[t] = t + 1 < n ? -(et * lay[t + 1]) / (et + lay[t + 1]) : 0.0;
    const double sn = sin(M_PI * (t + 1) / (2.0 * n));
    lam[t] = 2.0 * sn * sn;
  }
  for (int x = threadIdx.x; x < nn; x += blockDim.x) q[x] = dst2(n, x / n + 1, x % n);
  __syncthreads();
  // the two perpendicular axes in increasing order: node (t, u, v)
  const int pa = axis == 0 ? 1 : 0, qa = axis == 2 ? 1 : 2;
  const int c = (n - 1) / 2;
  double* Z = scratch + static_cast<size_t>(key) * 8 * m;  // [4][k1][k2][t]
  double* Wb = Z + 4 * static_cast<size_t>(m);              // [4][k1][t][v]
  // right-hand sides (sgf.cpp:243, :265-283): unit vectors at nodes given
  // in global (x, y, z) coordinates, mapped to (t, u, v)
  struct Term {
    int t, u, v;
    double s;
  };
  auto rhs_terms = [&](int r, Term* T, double* denom) -> int {
    int cen[3] = {c, c, c};
    if (r == 0) {
      T[0] = {c, c, c, 1.0};
      *denom = 1.0;
      return 1;
    }
    const int g = r - 1;
    const bool up = c + 1 < n, dn = c - 1 >= 0;
    int pl[3] = {cen[0], cen[1], cen[2]}, mi[3] = {cen[0], cen[1], cen[2]};
    if (up && dn) {
      pl[g] += 1;
      mi[g] -= 1;
      *denom = 2.0;  // 2 * unit pitch
    } else if (up) {
      pl[g] += 1;
      *denom = 1.0;
    } else if (dn) {
      mi[g] -= 1;
      *denom = 1.0;
    } else {
      return 0;  // n = 1: zero kernel
    }
    T[0] = {pl[axis], pl[pa], pl[qa], 1.0};
    T[1] = {mi[axis], mi[pa], mi[qa], -1.0};
    return 2;
  };
  // 1) one tridiagonal solve per (rhs, mode)
  for (int job = threadIdx.x; job < 4 * nn; job += blockDim.x) {
    const int r = job / nn, k1 = (job % nn) / n, k2 = job % n;
    Term T[2];
    double denom;
    const int nt = rhs_terms(r, T, &denom);
    double* z = Z + (static_cast<size_t>(r) * nn + k1 * n + k2) * n;
    double beta[kMaxN];
    for (int t = 0; t < n; ++t) beta[t] = 0.0;
    for (int a = 0; a < nt; ++a) beta[T[a].t] += T[a].s * q[k1 * n + T[a].u] * q[k2 * n + T[a].v];
    const double lm = lam[k1] + lam[k2];
    // Thomas algorithm on (A + lm E), symmetric positive definite
    double cp[kMaxN];
    double d0 = adiag[0] + lm * e[0];
    cp[0] = aoff[0] / d0;
    z[0] = beta[0] / d0;
    for (int t = 1; t < n; ++t) {
      const double d = adiag[t] + lm * e[t] - aoff[t - 1] * cp[t - 1];
      cp[t] = aoff[t] / d;
      z[t] = (beta[t] - aoff[t - 1] * z[t - 1]) / d;
    }
    for (int t = n - 2; t >= 0; --t) z[t] -= cp[t] * z[t + 1];
  }
  __syncthreads();
  // 2) W[r][k1][t][v] = sum_k2 q_k2[v] Z[r][k1][k2][t]
  for (int x = threadIdx.x; x < 4 * m; x += blockDim.x) {
    const int r = x / m, rem = x % m;
    const int k1 = rem / nn, t = (rem / n) % n, v = rem % n;
    const double* z = Z + (static_cast<size_t>(r) * nn + k1 * n) * n + t;
    double acc = 0;
    for (int k2 = 0; k2 < n; ++k2) acc += q[k2 * n + v] * z[static_cast<size_t>(k2) * n];
    Wb[x] = acc;
  }
  __syncthreads();
  // 3) boundary values z(t,u,v) = sum_k1 q_k1[u] W[k1][t][v]; panel outputs
  //    y = e_t z (A_IB^T (eps .* z)), panel = (face*n + w)*n + u (sgf.hpp:34-36)
  for (int x = threadIdx.x; x < 4 * P; x += blockDim.x) {
    const int r = x / P, pq = x % P;
    Term T[2];
    double denom;
    const int nt = rhs_terms(r, T, &denom);
    double* o = out + (static_cast<size_t>(key) * 4 + r) * P;
    if (nt == 0) {
      o[pq] = 0.0;
      continue;
    }
    const int face = pq / nn, rem = pq - face * nn;
    const int pu = rem % n, pw = rem / n;
    const int fa = face >> 1;
    int ci[3];
    ci[fa] = (face & 1) ? n - 1 : 0;
    ci[fa == 0 ? 1 : 0] = pu;
    ci[fa == 2 ? 1 : 2] = pw;
    const int t = ci[axis], u = ci[pa], v = ci[qa];
    const double* w = Wb + static_cast<size_t>(r) * m;
    double acc = 0;
    for (int k1 = 0; k1 < n; ++k1) acc += q[k1 * n + u] * w[(k1 * n + t) * n + v];
    o[pq] = e[t] * acc / denom;
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
    return frw_fail(ctx, FRW_EINVAL, "sgf_solve: need 1 <= n <= 128");
  if (count == 0) return FRW_OK;
  for (int q = 0; q < count; ++q)
    if (axes[q] < 0 || axes[q] > 2) return frw_fail(ctx, FRW_EINVAL, "sgf_solve: bad axis");
  FRW_CUDA(ctx, cudaSetDevice(ctx->device));
  const size_t m = static_cast<size_t>(n) * n * n, P = 6ull * n * n;
  // bounded scratch (kept in the context): solve in chunks of keys, at most
  // 128 keys or ~2 GB of slabs (8 n^3 doubles per key: 134 MB at n = 128)
  const int chunk = static_cast<int>(std::max<size_t>(
      1, std::min<size_t>(std::min(count, 128), (size_t{2} << 30) / (64 * m))));
  const size_t b_lay = (8 * static_cast<size_t>(chunk) * n + 255) / 256 * 256;
  const size_t b_ax = (4 * static_cast<size_t>(chunk) + 255) / 256 * 256;
  const size_t b_slab = 8 * 8 * m * static_cast<size_t>(chunk);
  const size_t b_out = 8 * P * 4 * static_cast<size_t>(chunk);
  const size_t need = b_lay + b_ax + b_slab + b_out;
  if (ctx->solve_cap < need) {
    cudaFree(ctx->d_solve);
    ctx->d_solve = nullptr;
    ctx->solve_cap = 0;
    FRW_CUDA(ctx, cudaMalloc(&ctx->d_solve, need));
    ctx->solve_cap = need;
  }
  double* d_lay = reinterpret_cast<double*>(ctx->d_solve);
  int* d_ax = reinterpret_cast<int*>(ctx->d_solve + b_lay);
  double* slab = reinterpret_cast<double*>(ctx->d_solve + b_lay + b_ax);
  double* out = reinterpret_cast<double*>(ctx->d_solve + b_lay + b_ax + b_slab);
  std::vector<double> h(P * 4 * static_cast<size_t>(chunk));
  int rc = FRW_OK;
  for (int k0 = 0; k0 < count && rc == FRW_OK; k0 += chunk) {
    const int kc = std::min(chunk, count - k0);
    cudaMemcpyAsync(d_lay, layers + static_cast<size_t>(k0) * n, 8 * static_cast<size_t>(kc) * n,
                    cudaMemcpyHostToDevice, ctx->stream);
    cudaMemcpyAsync(d_ax, axes + k0, 4 * static_cast<size_t>(kc), cudaMemcpyHostToDevice,
                    ctx->stream);
    const int qbytes = 8 * n * n;  // the DST-II basis (128 KB at n = 128)
    if (qbytes > 48 * 1024)
      cudaFuncSetAttribute(k_sgf_direct, cudaFuncAttributeMaxDynamicSharedMemorySize, qbytes);
    k_sgf_direct<<<kc, kDirectThreads, qbytes, ctx->stream>>>(n, d_ax, d_lay, slab, out);
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
  return rc;
}

extern "C" int frw_grid_sgf_solve(frw_ctx* ctx, int n, int count, const double* eps,
                                  double half_width, double* probs, double* kernels,
                                  double* steps) {
  if (!ctx || !eps || (!probs && !kernels && !steps)) return FRW_EINVAL;
  if (n < 1 || n > kGridMaxN || count < 0 || !(half_width > 0))
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
