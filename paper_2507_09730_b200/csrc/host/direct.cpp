// direct.cpp -- host direct solves of the transition-cube system.
//
// The reference solves s_ii z = b by Jacobi-PCG and falls back to a sparse
// LDL^T factorisation (SimplicialLDLT) when the iteration stalls
// (sgf.cpp:162-211); its oracle cross-checks the surface Green's function
// against a dense LU of the absorption matrix (oracle.cpp:15-92,
// exact_absorption_row).  The device build solves stratified keys exactly
// (sgf_solve.cu, k_sgf_direct) and general grids by device Jacobi-PCG
// (k_grid_pcg); this file holds the host counterparts of the two direct
// paths:
//
//  * direct_sgf: s_ii in band form (natural node order, half bandwidth
//    <= n^2) factored as L D L^T, probabilities, gradient kernels and the
//    expected step count of a grid -- masked (conductor-voxel) grids
//    included, with the conductor panels appended in (node, direction)
//    order (sgf.cpp:94-118).  solve_sgf uses it for masked grids and when
//    the device PCG does not converge.  O(n^7) work: n <= kDirectMaxN.
//  * exact_absorption_row: the dense LU row of a_ii^{-1} a_ib at the start
//    node, assembled independently of the band system (validate-sgf's
//    n <= 6 cross-check, cli.cpp:271-279).
#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <vector>

#include "frwcap.hpp"

namespace frwcap {

namespace {

constexpr int kDirectMaxN = 32;

// one lattice step per direction d = 2 * axis + (positive ? 1 : 0)
inline void step_of(int dir, int* di, int* dj, int* dk) {
  const int s = (dir & 1) ? 1 : -1, a = dir >> 1;
  *di = a == 0 ? s : 0;
  *dj = a == 1 ? s : 0;
  *dk = a == 2 ? s : 0;
}

// surface panel of the face a node steps out of (sgf.cpp:13-30)
inline int surface_panel(int n, int i, int j, int k, int dir) {
  const int a = dir >> 1;
  const int u = a == 0 ? j : i;
  const int v = a == 2 ? j : k;
  return (dir * n + v) * n + u;
}

struct BandSystem {
  int n = 0, rows = 0, bw = 0, panels = 0, center = -1;
  std::vector<int> row_of, node_of;
  std::vector<double> eps, rsum;          // per row
  std::vector<int> absorb;                // [rows][6] panel index or -1
  std::vector<double> L;                  // unit lower band, [rows][bw]: L(r, r - 1 - q)
  std::vector<double> D;                  // diagonal of L D L^T
  std::vector<double> off;                // s_ii lower band before factoring (same layout)

  double& band(std::vector<double>& b, int r, int c) { return b[static_cast<size_t>(r) * bw + (r - 1 - c)]; }

  explicit BandSystem(const DielectricGrid& g) {
    n = g.n;
    const int nvox = n * n * n;
    if (n < 1 || static_cast<int>(g.eps.size()) != nvox)
      throw std::invalid_argument("direct solve: malformed grid");
    const bool masked = g.has_mask();
    row_of.assign(nvox, -1);
    for (int idx = 0; idx < nvox; ++idx)
      if (!masked || g.conductor_mask[idx] < 0) {
        row_of[idx] = static_cast<int>(node_of.size());
        node_of.push_back(idx);
      }
    rows = static_cast<int>(node_of.size());
    if (rows == 0) throw std::invalid_argument("direct solve: no interior nodes");
    const int c = (n - 1) / 2;  // start_node (sgf.hpp:58-61)
    center = row_of[(c * n + c) * n + c];
    if (center < 0) throw std::invalid_argument("direct solve: start node is masked");
    // half bandwidth: the largest row distance of two neighbouring rows
    bw = 1;
    for (int r = 0; r < rows; ++r) {
      const int idx = node_of[r];
      const int i = idx % n, j = (idx / n) % n, k = idx / (n * n);
      for (int dir = 0; dir < 6; dir += 2) {  // lower neighbours only
        int di, dj, dk;
        step_of(dir, &di, &dj, &dk);
        const int ni = i + di, nj = j + dj, nk = k + dk;
        if (ni < 0 || nj < 0 || nk < 0) continue;
        const int nr = row_of[(nk * n + nj) * n + ni];
        if (nr >= 0) bw = std::max(bw, r - nr);
      }
    }
    eps.resize(rows);
    rsum.assign(rows, 0.0);
    absorb.assign(static_cast<size_t>(rows) * 6, -1);
    off.assign(static_cast<size_t>(rows) * bw, 0.0);
    D.assign(rows, 0.0);
    panels = 6 * n * n;
    for (int r = 0; r < rows; ++r) {
      const int idx = node_of[r];
      const int i = idx % n, j = (idx / n) % n, k = idx / (n * n);
      const double ev = g.eps[idx];
      eps[r] = ev;
      double row_sum = 0;
      for (int dir = 0; dir < 6; ++dir) {
        int di, dj, dk;
        step_of(dir, &di, &dj, &dk);
        const int ni = i + di, nj = j + dj, nk = k + dk;
        if (ni < 0 || ni >= n || nj < 0 || nj >= n || nk < 0 || nk >= n) {
          absorb[static_cast<size_t>(r) * 6 + dir] = surface_panel(n, i, j, k, dir);
          row_sum += 1.0;
          continue;
        }
        const int nr = row_of[(nk * n + nj) * n + ni];
        if (nr < 0) {  // conductor voxel: an absorbing panel of its own
          absorb[static_cast<size_t>(r) * 6 + dir] = panels++;
          row_sum += 1.0;
          continue;
        }
        const double ei = g.eps[(nk * n + nj) * n + ni];
        row_sum += ei / (ei + ev);
        if (nr < r) band(off, r, nr) = -(ev * ei) / (ev + ei);
      }
      rsum[r] = row_sum;
      D[r] = ev * row_sum;
    }
    factor();
  }

  // s_ii = L D L^T in place (band Crout, row by row)
  void factor() {
    L = off;
    std::vector<double> w(bw);
    for (int r = 0; r < rows; ++r) {
      const int c0 = std::max(0, r - bw);
      // w[c] = L(r, c) D(c) for c in [c0, r), built left to right
      for (int c = c0; c < r; ++c) {
        double s = band(off, r, c);
        const int k0 = std::max(c0, c - bw);
        for (int k = k0; k < c; ++k) s -= band(L, r, k) * D[k] * band(L, c, k);
        band(L, r, c) = s / D[c];
      }
      double d = D[r];
      for (int c = c0; c < r; ++c) d -= band(L, r, c) * band(L, r, c) * D[c];
      if (!(d > 0)) throw SolveError("transition cube solve failed: factorization error", 0.0);
      D[r] = d;
    }
  }

  // z = s_ii^{-1} b
  std::vector<double> solve(std::vector<double> z) {
    for (int r = 0; r < rows; ++r)
      for (int c = std::max(0, r - bw); c < r; ++c) z[r] -= band(L, r, c) * z[c];
    for (int r = 0; r < rows; ++r) z[r] /= D[r];
    for (int r = rows - 1; r >= 0; --r)
      for (int q = r + 1; q <= std::min(rows - 1, r + bw); ++q) z[r] -= band(L, q, r) * z[q];
    return z;
  }

  // a_ib^T (eps .* s_ii^{-1} b): the absorption row of right-hand side b
  std::vector<double> panels_of(const std::vector<double>& b) {
    const std::vector<double> z = solve(b);
    std::vector<double> p(panels, 0.0);
    for (int r = 0; r < rows; ++r)
      for (int dir = 0; dir < 6; ++dir) {
        const int pa = absorb[static_cast<size_t>(r) * 6 + dir];
        if (pa >= 0) p[pa] += eps[r] * z[r];
      }
    return p;
  }
};

}  // namespace

DirectSgf direct_sgf(const DielectricGrid& g, bool with_kernels) {
  if (g.n > kDirectMaxN)
    throw std::invalid_argument("direct solve: n exceeds the host band-solver cap (32)");
  BandSystem S(g);
  DirectSgf out;
  DiscreteSGF& sgf = out.sgf;
  sgf.n = g.n;
  sgf.pitch = g.pitch();
  std::vector<double> e(S.rows, 0.0);
  e[S.center] = 1.0;
  const std::vector<double> p = S.panels_of(e);
  double sum = 0, lo = 0;
  for (double v : p) {
    sum += v;
    lo = std::min(lo, v);
  }
  if (std::fabs(sum - 1.0) > 1e-9 || lo < -1e-9)  // sgf.cpp:249-253
    throw SolveError("transition cube solve failed normalization check", std::fabs(sum - 1.0));
  sgf.probs.resize(p.size());
  sgf.cdf.resize(p.size());
  double run = 0;
  for (size_t b = 0; b < p.size(); ++b) {
    sgf.probs[b] = std::max(p[b], 0.0);
    sgf.cdf[b] = run += sgf.probs[b];
  }
  if (with_kernels) {  // sgf.cpp:268-296: central difference at the start node
    const int n = g.n, c = (n - 1) / 2;
    for (int axis = 0; axis < 3; ++axis) {
      auto nb_row = [&](int delta) {
        int v[3] = {c, c, c};
        v[axis] += delta;
        if (v[axis] < 0 || v[axis] >= n) return -1;
        return S.row_of[(v[2] * n + v[1]) * n + v[0]];
      };
      const int rp = nb_row(+1), rm = nb_row(-1);
      auto& kernel = sgf.grad_kernels[axis];
      kernel.assign(p.size(), 0.0);
      std::vector<double> rhs(S.rows, 0.0);
      double denom;
      if (rp >= 0 && rm >= 0) {
        rhs[rp] += 1.0;
        rhs[rm] -= 1.0;
        denom = 2.0 * sgf.pitch;
      } else if (rp >= 0) {
        rhs[rp] += 1.0;
        rhs[S.center] -= 1.0;
        denom = sgf.pitch;
      } else if (rm >= 0) {
        rhs[S.center] += 1.0;
        rhs[rm] -= 1.0;
        denom = sgf.pitch;
      } else {
        continue;  // n = 1: no interior neighbours, zero kernel
      }
      const std::vector<double> row = S.panels_of(rhs);
      for (size_t b = 0; b < row.size(); ++b) kernel[b] = row[b] / denom;
    }
  }
  // expected steps: a_ii t = rowsum  <=>  s_ii t = eps .* rowsum (sgf.cpp:292-299)
  std::vector<double> b(S.rows);
  for (int r = 0; r < S.rows; ++r) b[r] = S.eps[r] * S.rsum[r];
  out.expected_steps = S.solve(b)[S.center];
  return out;
}

// Dense LU of a_ii^T, an assembly independent of BandSystem (oracle.cpp:15-92)
std::vector<double> exact_absorption_row(const DielectricGrid& grid, int cap) {
  const int n = grid.n;
  if (n > cap) throw std::invalid_argument("exact_absorption_row: n exceeds cost cap");
  const int nvox = n * n * n;
  std::vector<int> row(nvox, -1), node;
  for (int idx = 0; idx < nvox; ++idx)
    if (!grid.has_mask() || grid.conductor_mask[idx] < 0) {
      row[idx] = static_cast<int>(node.size());
      node.push_back(idx);
    }
  const int R = static_cast<int>(node.size());
  if (R == 0) throw std::invalid_argument("grid has no interior nodes");
  // panels: 6 n^2 surface panels, then conductor panels in (node, direction) order
  int panels = 6 * n * n;
  std::vector<int> cpanel(static_cast<size_t>(nvox) * 6, -1);
  for (int r = 0; r < R; ++r) {
    const int idx = node[r], i = idx % n, j = (idx / n) % n, k = idx / (n * n);
    for (int dir = 0; dir < 6; ++dir) {
      int di, dj, dk;
      step_of(dir, &di, &dj, &dk);
      const int ni = i + di, nj = j + dj, nk = k + dk;
      if (ni < 0 || ni >= n || nj < 0 || nj >= n || nk < 0 || nk >= n) continue;
      if (row[(nk * n + nj) * n + ni] < 0) cpanel[static_cast<size_t>(idx) * 6 + dir] = panels++;
    }
  }
  // At = a_ii^T (dense, row-major), Bp[r] = the absorbing panels of row r
  std::vector<double> At(static_cast<size_t>(R) * R, 0.0);
  std::vector<std::vector<int>> Bp(R);
  for (int r = 0; r < R; ++r) {
    const int idx = node[r], i = idx % n, j = (idx / n) % n, k = idx / (n * n);
    const double ev = grid.eps[idx];
    double diag = 0;
    for (int dir = 0; dir < 6; ++dir) {
      int di, dj, dk;
      step_of(dir, &di, &dj, &dk);
      const int ni = i + di, nj = j + dj, nk = k + dk;
      if (ni < 0 || ni >= n || nj < 0 || nj >= n || nk < 0 || nk >= n) {
        Bp[r].push_back(surface_panel(n, i, j, k, dir));
        diag += 1.0;
        continue;
      }
      const int nidx = (nk * n + nj) * n + ni;
      if (row[nidx] < 0) {
        Bp[r].push_back(cpanel[static_cast<size_t>(idx) * 6 + dir]);
        diag += 1.0;
        continue;
      }
      const double a = grid.eps[nidx] / (grid.eps[nidx] + ev);
      At[static_cast<size_t>(row[nidx]) * R + r] -= a;  // a_ii(r, nb) into At(nb, r)
      diag += a;
    }
    At[static_cast<size_t>(r) * R + r] = diag;
  }
  const int c = (n - 1) / 2;
  const int crow = row[(c * n + c) * n + c];
  if (crow < 0) throw std::invalid_argument("start node is masked");
  // solve At y = e_c by Gaussian elimination with partial pivoting
  std::vector<double> y(R, 0.0);
  y[crow] = 1.0;
  for (int col = 0; col < R; ++col) {
    int piv = col;
    for (int r = col + 1; r < R; ++r)
      if (std::fabs(At[static_cast<size_t>(r) * R + col]) > std::fabs(At[static_cast<size_t>(piv) * R + col]))
        piv = r;
    if (piv != col) {
      for (int q = 0; q < R; ++q)
        std::swap(At[static_cast<size_t>(col) * R + q], At[static_cast<size_t>(piv) * R + q]);
      std::swap(y[col], y[piv]);
    }
    const double d = At[static_cast<size_t>(col) * R + col];
    if (d == 0) throw std::runtime_error("exact_absorption_row: singular system");
    for (int r = col + 1; r < R; ++r) {
      const double f = At[static_cast<size_t>(r) * R + col] / d;
      if (f == 0) continue;
      for (int q = col; q < R; ++q) At[static_cast<size_t>(r) * R + q] -= f * At[static_cast<size_t>(col) * R + q];
      y[r] -= f * y[col];
    }
  }
  for (int r = R - 1; r >= 0; --r) {
    double s = y[r];
    for (int q = r + 1; q < R; ++q) s -= At[static_cast<size_t>(r) * R + q] * y[q];
    y[r] = s / At[static_cast<size_t>(r) * R + r];
  }
  std::vector<double> p(panels, 0.0);
  for (int r = 0; r < R; ++r)
    for (int pa : Bp[r]) p[pa] += y[r];
  return p;
}

}  // namespace frwcap
