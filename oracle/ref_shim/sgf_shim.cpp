// sgf_shim.cpp -- TEST INFRASTRUCTURE: a restatement of the Eigen-dependent
// translation unit proj/src/sgf.cpp so the reference's remaining sources
// (microwalk.cpp, geometry.cpp, engine.cpp, sgf_cache.cpp) can be compiled
// unmodified into oracle/_ref/libfrwref.so (see oracle/Makefile).
//
// Restated symbols (declared in proj/include/frwcap/sgf.hpp):
//   surface_panel_of / decode_surface_panel / surface_panel_center /
//   surface_panel_offsets            sgf.cpp:13-55
//   assemble_system                  sgf.cpp:57-155
//   solve_sgf, expected_steps        sgf.cpp:162-299 (Jacobi-PCG on s_ii with
//                                    the adjoint trick; no LDLT fallback)
//   sample_panel                     sgf.cpp:301-308
// Differences: PCG dot products are scalar, so probabilities agree with an
// Eigen build to the solver tolerance (1e-10 rel), not bit for bit.
#include <algorithm>
#include <cmath>
#include <vector>

#include "frwcap/sgf.hpp"

namespace frwcap {

int surface_panel_of(int n, const Vec3i& voxel, int dir) {
  const int axis = kDirAxis[dir];
  const int u = axis == 0 ? voxel.y : voxel.x;
  const int v = axis == 2 ? voxel.y : voxel.z;
  return surface_panel_index(n, dir, u, v);
}

std::array<int, 3> decode_surface_panel(int n, int panel) {
  const int nn = n * n;
  return {panel / nn, (panel % nn) % n, (panel % nn) / n};
}

Vec3 surface_panel_center(const Cube& cube, int n, int panel) {
  const std::array<int, 3> fuv = decode_surface_panel(n, panel);
  const int axis = kDirAxis[fuv[0]];
  const double h = cube.half_width;
  const double pitch = 2.0 * h / n;
  const int b1 = axis == 0 ? 1 : 0;
  const int b2 = axis == 2 ? 1 : 2;
  Vec3 out;
  out[axis] = cube.center[axis] + kDirSign[fuv[0]] * h;
  out[b1] = cube.center[b1] - h + (fuv[1] + 0.5) * pitch;
  out[b2] = cube.center[b2] - h + (fuv[2] + 0.5) * pitch;
  return out;
}

std::array<double, 2> surface_panel_offsets(int n, int panel) {
  const std::array<int, 3> fuv = decode_surface_panel(n, panel);
  return {(fuv[1] + 0.5) * 2.0 / n - 1.0, (fuv[2] + 0.5) * 2.0 / n - 1.0};
}

FDSystem assemble_system(const DielectricGrid& grid) {
  const int n = grid.n;
  const int nvox = n * n * n;
  FDSystem sys;
  sys.n = n;
  sys.cube = grid.cube;
  sys.surface_panels = 6 * n * n;
  sys.row_of_node.assign(nvox, -1);
  for (int v = 0; v < nvox; ++v) {
    const bool free_voxel = !grid.has_mask() || grid.conductor_mask[v] < 0;
    if (!free_voxel) continue;
    sys.row_of_node[v] = static_cast<int32_t>(sys.node_of_row.size());
    sys.node_of_row.push_back(v);
  }
  const int rows = sys.interior_count();
  if (rows == 0) throw std::invalid_argument("assemble_system: no interior nodes");
  const Vec3i s = start_node(n);
  sys.center_row = sys.row_of_node[grid.index(s.x, s.y, s.z)];
  if (sys.center_row < 0)
    throw std::invalid_argument("assemble_system: start node is masked");

  for (int p = 0; p < sys.surface_panels; ++p) {
    PanelInfo pi;
    pi.center = surface_panel_center(grid.cube, n, p);
    pi.face = static_cast<int8_t>(p / (n * n));
    sys.panels.push_back(pi);
  }
  sys.eps_interior.resize(rows);
  sys.alpha_row_sum.resize(rows);

  using T = Eigen::Triplet<double>;
  std::vector<T> aii, sii, aib;
  const double pitch = grid.pitch();
  for (int v = 0; v < nvox; ++v) {
    const int r = sys.row_of_node[v];
    if (r < 0) continue;
    const Vec3i c{v % n, (v / n) % n, v / (n * n)};
    const double ev = grid.eps[v];
    sys.eps_interior[r] = ev;
    double diag = 0;
    for (int d = 0; d < 6; ++d) {
      Vec3i nb = c;
      nb[kDirAxis[d]] += kDirSign[d];
      const int ax = kDirAxis[d];
      if (nb[ax] < 0 || nb[ax] >= n) {
        aib.emplace_back(r, surface_panel_of(n, c, d), 1.0);
        diag += 1.0;
        continue;
      }
      const int nv = grid.index(nb.x, nb.y, nb.z);
      const int nr = sys.row_of_node[nv];
      if (nr < 0) {
        // absorbing conductor face, appended after the surface panels
        PanelInfo pi;
        pi.center = grid.voxel_center(c.x, c.y, c.z);
        pi.center[ax] += kDirSign[d] * pitch / 2;
        pi.conductor = grid.conductor_mask[nv];
        pi.face = static_cast<int8_t>(d);
        aib.emplace_back(r, static_cast<int>(sys.panels.size()), 1.0);
        sys.panels.push_back(pi);
        diag += 1.0;
        continue;
      }
      const double ei = grid.eps[nv];
      aii.emplace_back(r, nr, -(ei / (ei + ev)));
      sii.emplace_back(r, nr, -(ev * ei) / (ev + ei));
      diag += ei / (ei + ev);
    }
    aii.emplace_back(r, r, diag);
    sii.emplace_back(r, r, ev * diag);
    sys.alpha_row_sum[r] = diag;
  }
  sys.a_ii.resize(rows, rows);
  sys.a_ii.setFromTriplets(aii.begin(), aii.end());
  sys.s_ii.resize(rows, rows);
  sys.s_ii.setFromTriplets(sii.begin(), sii.end());
  sys.a_ib.resize(rows, sys.panel_count());
  sys.a_ib.setFromTriplets(aib.begin(), aib.end());
  return sys;
}

namespace {

using Vec = std::vector<double>;

void spmv(const Eigen::SparseMatrix<double>& A, const Vec& x, Vec& y) {
  const auto& ptr = A.outer();
  const auto& col = A.inner();
  const auto& val = A.values();
  for (Eigen::Index r = 0; r < A.rows(); ++r) {
    double acc = 0;
    for (Eigen::Index i = ptr[r]; i < ptr[r + 1]; ++i) acc += val[i] * x[col[i]];
    y[r] = acc;
  }
}

double dotp(const Vec& a, const Vec& b) {
  double s = 0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

// Jacobi-preconditioned CG from a zero guess; converged when
// |r|^2 < tol^2 |b|^2 within factor*rows iterations.
Vec pcg(const FDSystem& sys, const Vec& b, const SolverOptions& o) {
  const size_t m = b.size();
  Vec inv(m), x(m, 0.0), r = b, z(m), p(m), t(m);
  const auto& ptr = sys.s_ii.outer();
  const auto& col = sys.s_ii.inner();
  const auto& val = sys.s_ii.values();
  for (size_t i = 0; i < m; ++i) {
    double dg = 0;
    for (Eigen::Index k = ptr[i]; k < ptr[i + 1]; ++k)
      if (col[k] == Eigen::Index(i)) dg = val[k];
    inv[i] = dg != 0 ? 1.0 / dg : 1.0;
  }
  const double b2 = dotp(b, b);
  if (b2 == 0) return x;
  const double thr = o.rel_tol * o.rel_tol * b2;
  if (dotp(r, r) < thr) return x;
  for (size_t i = 0; i < m; ++i) p[i] = inv[i] * r[i];
  double rz = dotp(r, p);
  const long cap = static_cast<long>(o.max_iter_factor) * static_cast<long>(m);
  for (long it = 0; it < cap; ++it) {
    spmv(sys.s_ii, p, t);
    const double a = rz / dotp(p, t);
    for (size_t i = 0; i < m; ++i) {
      x[i] += a * p[i];
      r[i] -= a * t[i];
    }
    const double rr = dotp(r, r);
    if (rr < thr) return x;
    for (size_t i = 0; i < m; ++i) z[i] = inv[i] * r[i];
    const double rz_old = rz;
    rz = dotp(r, z);
    for (size_t i = 0; i < m; ++i) p[i] = z[i] + (rz / rz_old) * p[i];
  }
  throw SolveError("transition cube solve failed: PCG did not converge",
                   std::sqrt(dotp(r, r) / b2));
}

// a_ib^T (eps .* z)
Vec boundary_row(const FDSystem& sys, const Vec& z) {
  Vec out(sys.panel_count(), 0.0);
  const auto& ptr = sys.a_ib.outer();
  const auto& col = sys.a_ib.inner();
  const auto& val = sys.a_ib.values();
  for (Eigen::Index r = 0; r < sys.a_ib.rows(); ++r) {
    const double y = sys.eps_interior[r] * z[r];
    for (Eigen::Index i = ptr[r]; i < ptr[r + 1]; ++i) out[col[i]] += val[i] * y;
  }
  return out;
}

int row_at(const FDSystem& sys, int axis, int delta) {
  Vec3i c = start_node(sys.n);
  c[axis] += delta;
  if (c[axis] < 0 || c[axis] >= sys.n) return -1;
  return sys.row_of_node[(c.z * sys.n + c.y) * sys.n + c.x];
}

}  // namespace

DiscreteSGF solve_sgf(const FDSystem& sys, bool with_kernels,
                      const SolverOptions& opts) {
  const int rows = sys.interior_count();
  const int panels = sys.panel_count();
  DiscreteSGF out;
  out.n = sys.n;
  out.pitch = 2.0 * sys.cube.half_width / sys.n;
  out.surface_panels = sys.surface_panels;

  Vec e(rows, 0.0);
  e[sys.center_row] = 1.0;
  const Vec p = boundary_row(sys, pcg(sys, e, opts));
  double total = 0, lowest = 0;
  for (double v : p) {
    total += v;
    lowest = std::min(lowest, v);
  }
  if (std::abs(total - 1.0) > 1e-9 || lowest < -1e-9)
    throw SolveError("transition cube solve failed normalization check",
                     std::abs(total - 1.0));
  out.probs.resize(panels);
  out.cdf.resize(panels);
  double run = 0;
  for (int b = 0; b < panels; ++b) {
    out.probs[b] = std::max(p[b], 0.0);
    run += out.probs[b];
    out.cdf[b] = run;
  }
  if (!with_kernels) return out;
  for (int axis = 0; axis < 3; ++axis) {
    out.grad_kernels[axis].assign(panels, 0.0);
    const int up = row_at(sys, axis, +1), dn = row_at(sys, axis, -1);
    Vec rhs(rows, 0.0);
    double denom;
    if (up >= 0 && dn >= 0) {
      rhs[up] += 1.0;
      rhs[dn] -= 1.0;
      denom = 2.0 * out.pitch;
    } else if (up >= 0) {
      rhs[up] += 1.0;
      rhs[sys.center_row] -= 1.0;
      denom = out.pitch;
    } else if (dn >= 0) {
      rhs[sys.center_row] += 1.0;
      rhs[dn] -= 1.0;
      denom = out.pitch;
    } else {
      continue;
    }
    const Vec k = boundary_row(sys, pcg(sys, rhs, opts));
    for (int b = 0; b < panels; ++b) out.grad_kernels[axis][b] = k[b] / denom;
  }
  return out;
}

double expected_steps(const FDSystem& sys, const SolverOptions& opts) {
  Vec rhs(sys.interior_count());
  for (int r = 0; r < sys.interior_count(); ++r)
    rhs[r] = sys.eps_interior[r] * sys.alpha_row_sum[r];
  return pcg(sys, rhs, opts)[sys.center_row];
}

int sample_panel(const DiscreteSGF& sgf, double u) {
  const double target = u * sgf.cdf.back();
  const auto it = std::upper_bound(sgf.cdf.begin(), sgf.cdf.end(), target);
  if (it == sgf.cdf.end()) return static_cast<int>(sgf.cdf.size()) - 1;
  return static_cast<int>(it - sgf.cdf.begin());
}

}  // namespace frwcap
