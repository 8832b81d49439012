// microwalk.cpp -- the reference's single-transit MicroWalk API on the device.
//
// Mirrors proj/include/frwcap/microwalk.hpp:18-100 and sgf.hpp:24-61: Exit,
// EngulfedStart, neighbor_weights, microwalk_transit (materialised grid),
// microwalk_transit_lazy and microwalk_e_transit (structure cubes), plus the
// lattice/panel algebra and build_grid/classify_grid (geometry.cpp:264-349).
// Transits run on the device through the C ABI: grid transits through
// frw_microwalk_batch in FRW_RNG_SPLITMIX_STATES mode, structure transits
// through frw_structure_transits; the caller's SplitMix64 is continued
// exactly (its raw state goes in, state + steps * gamma comes out), so
// results are bit-identical to the reference for the same stream.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>

#include "frwcap.hpp"

namespace frwcap {

namespace {
constexpr double kEpsRelTol = 1e-9;  // geometry.cpp:14

// FNV-style fingerprint over 64-bit words (then the tail bytes)
uint64_t fnv(uint64_t h, const void* p, size_t n) {
  const auto* b = static_cast<const unsigned char*>(p);
  size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    uint64_t w;
    std::memcpy(&w, b + i, 8);
    h = (h ^ w) * 0x100000001B3ull;
    h ^= h >> 29;
  }
  for (; i < n; ++i) h = (h ^ b[i]) * 0x100000001B3ull;
  return h;
}

std::mutex g_mu;
// fingerprint of the grid / structure each context holds
std::map<frw_ctx*, uint64_t>& grid_fp() {
  static auto* m = new std::map<frw_ctx*, uint64_t>;
  return *m;
}
std::map<frw_ctx*, uint64_t>& structure_fp() {
  static auto* m = new std::map<frw_ctx*, uint64_t>;
  return *m;
}

void ensure_grid(frw_ctx* ctx, const DielectricGrid& g) {
  const size_t nodes = static_cast<size_t>(g.n) * g.n * g.n;
  if (g.n < 1 || g.eps.size() != nodes || (g.has_mask() && g.conductor_mask.size() != nodes))
    throw std::invalid_argument("microwalk_transit: malformed DielectricGrid");
  uint64_t h = 0xcbf29ce484222325ull;
  h = fnv(h, &g.n, sizeof g.n);
  h = fnv(h, &g.cube, sizeof g.cube);
  h = fnv(h, g.eps.data(), 8 * nodes);
  if (g.has_mask()) h = fnv(h, g.conductor_mask.data(), 4 * nodes);
  h |= 1;
  std::lock_guard<std::mutex> lk(g_mu);
  if (grid_fp()[ctx] == h) return;
  throw_status(ctx, frw_upload_grid(ctx, g.n, g.eps.data(),
                                    g.has_mask() ? g.conductor_mask.data() : nullptr,
                                    g.cube.center.x, g.cube.center.y, g.cube.center.z,
                                    g.cube.half_width));
  grid_fp()[ctx] = h;
}

Vec3 voxel_center(const Cube& cube, int n, const Vec3i& v) {  // microwalk.cpp:24-30
  const double h = cube.half_width, p = 2.0 * h / n;
  return {cube.center.x - h + (v.x + 0.5) * p, cube.center.y - h + (v.y + 0.5) * p,
          cube.center.z - h + (v.z + 0.5) * p};
}

Exit exit_from_grid(const DielectricGrid& g, int32_t panel, int32_t steps, int32_t cond,
                    int64_t nd) {
  const int n = g.n;
  Exit e;
  e.steps = steps;
  const int64_t idx = nd >> 3;
  e.dir = static_cast<int>(nd & 7);
  e.voxel = {static_cast<int>(idx % n), static_cast<int>((idx / n) % n),
             static_cast<int>(idx / (static_cast<int64_t>(n) * n))};
  if (panel >= 0) {
    e.kind = Exit::Kind::Surface;
    e.panel = panel;
    e.point = surface_panel_center(g.cube, n, panel);
  } else {
    e.kind = Exit::Kind::Conductor;
    e.conductor_id = cond;
    Vec3 p = voxel_center(g.cube, n, e.voxel);
    p[kDirAxis[e.dir]] += kDirSign[e.dir] * g.cube.half_width / n;  // microwalk.cpp:141-143
    e.point = p;
  }
  return e;
}
}  // namespace

bool eps_equal(double a, double b) {
  return std::abs(a - b) <= kEpsRelTol * std::max(std::abs(a), std::abs(b));
}

FreeCube Structure::max_free_cube(const Vec3& p) const {  // geometry.cpp:64-80
  FreeCube r;
  r.half_width = world.chebyshev_to_wall(p);
  if (r.half_width <= 0) throw std::invalid_argument("max_free_cube: point not inside the world");
  for (const auto& c : conductors) {
    const double d = c.box.chebyshev_to(p);
    if (d <= 0)
      throw std::invalid_argument("max_free_cube: point inside conductor " +
                                  std::to_string(c.id));
    if (d <= r.half_width) {  // ties go to the conductor
      r.half_width = d;
      r.nearest_id = c.id;
    }
  }
  return r;
}

// ---- lattice and panel algebra (sgf.cpp:13-55) ----------------------------------
int surface_panel_of(int n, const Vec3i& voxel, int dir) {
  const int a = kDirAxis[dir];
  const int u = a == 0 ? voxel.y : voxel.x;
  const int v = a == 2 ? voxel.y : voxel.z;
  return surface_panel_index(n, dir, u, v);
}

std::array<int, 3> decode_surface_panel(int n, int panel) {
  const int face = panel / (n * n);
  const int rem = panel % (n * n);
  return {face, rem % n, rem / n};
}

Vec3 surface_panel_center(const Cube& cube, int n, int panel) {
  const auto [face, u, v] = decode_surface_panel(n, panel);
  const int axis = kDirAxis[face];
  const double h = cube.half_width, pitch = 2.0 * h / n;
  Vec3 p;
  p[axis] = cube.center[axis] + kDirSign[face] * h;
  const int b1 = axis == 0 ? 1 : 0;
  const int b2 = axis == 2 ? 1 : 2;
  p[b1] = cube.center[b1] - h + (u + 0.5) * pitch;
  p[b2] = cube.center[b2] - h + (v + 0.5) * pitch;
  return p;
}

std::array<double, 2> surface_panel_offsets(int n, int panel) {
  const auto [face, u, v] = decode_surface_panel(n, panel);
  (void)face;
  return {(u + 0.5) * 2.0 / n - 1.0, (v + 0.5) * 2.0 / n - 1.0};
}

// ---- voxelisation (geometry.cpp:264-349) ---------------------------------------
void classify_grid(DielectricGrid& g) {
  const int n = g.n;
  double ref = -1;
  bool uniform = true;
  for (int k = 0; k < n && uniform; ++k)
    for (int j = 0; j < n && uniform; ++j)
      for (int i = 0; i < n; ++i) {
        if (g.conductor(i, j, k) >= 0) continue;
        const double e = g.eps_at(i, j, k);
        if (ref < 0)
          ref = e;
        else if (!eps_equal(ref, e)) {
          uniform = false;
          break;
        }
      }
  if (uniform) {
    g.tag = GridTag::Uniform;
    g.strat_axis = -1;
    return;
  }
  for (int axis = 0; axis < 3; ++axis) {
    bool ok = true;
    for (int sl = 0; sl < n && ok; ++sl) {
      double slice_ref = -1;
      for (int u = 0; u < n && ok; ++u)
        for (int v = 0; v < n; ++v) {
          Vec3i c;
          c[axis] = sl;
          c[(axis + 1) % 3] = u;
          c[(axis + 2) % 3] = v;
          if (g.conductor(c.x, c.y, c.z) >= 0) continue;
          const double e = g.eps_at(c.x, c.y, c.z);
          if (slice_ref < 0)
            slice_ref = e;
          else if (!eps_equal(slice_ref, e)) {
            ok = false;
            break;
          }
        }
    }
    if (ok) {
      g.tag = GridTag::Stratified;
      g.strat_axis = axis;
      return;
    }
  }
  g.tag = GridTag::General;
  g.strat_axis = -1;
}

bool StratifiedProfile::uniform() const {
  return std::all_of(layers.begin(), layers.end(),
                     [&](double e) { return eps_equal(e, layers.front()); });
}

// geometry.cpp:357-396: the field inside the cube depends on one axis only
// when every dielectric meeting the OPEN cube spans the cube's cross-section
// perpendicular to it; the first such axis is read at the slice centres
std::optional<StratifiedProfile> stratified_profile(const Structure& s, const Cube& cube, int n) {
  const Box cb = cube.box();
  std::array<bool, 3> spans{true, true, true};
  bool met = false;
  for (const Dielectric& d : s.dielectrics) {
    if (!d.box.intersects_open(cb)) continue;
    met = true;
    for (int a = 0; a < 3; ++a)
      for (int b : {(a + 1) % 3, (a + 2) % 3})
        spans[a] = spans[a] && d.box.lo[b] <= cb.lo[b] && d.box.hi[b] >= cb.hi[b];
  }
  int axis = 0;  // the background alone: uniform
  if (met) {
    const auto it = std::find(spans.begin(), spans.end(), true);
    if (it == spans.end()) return std::nullopt;
    axis = static_cast<int>(it - spans.begin());
  }
  StratifiedProfile prof;
  prof.axis = axis;
  prof.layers.resize(n);
  const double pitch = 2.0 * cube.half_width / n;
  for (int t = 0; t < n; ++t) {
    Vec3 p = cube.center;
    p[axis] = cube.center[axis] - cube.half_width + (t + 0.5) * pitch;
    prof.layers[t] = s.permittivity_at(p);
  }
  if (prof.uniform()) prof.axis = 0;
  return prof;
}

DielectricGrid build_grid(const Structure& s, const Cube& cube, int n, bool allow_conductors) {
  if (n < 1) throw std::invalid_argument("build_grid: n must be >= 1");
  if (!s.world.contains_box(cube.box()))
    throw std::invalid_argument("build_grid: cube extends outside the world");
  DielectricGrid g;
  g.n = n;
  g.cube = cube;
  g.eps.resize(static_cast<size_t>(n) * n * n);
  if (allow_conductors) g.conductor_mask.assign(static_cast<size_t>(n) * n * n, -1);
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        const Vec3 p = g.voxel_center(i, j, k);
        g.eps[g.index(i, j, k)] = s.permittivity_at(p);
        const auto cid = s.conductor_at(p, 0.0);
        if (cid) {
          if (!allow_conductors)
            throw std::invalid_argument("build_grid: cube intersects conductor " +
                                        std::to_string(*cid));
          g.conductor_mask[g.index(i, j, k)] = *cid;
        }
      }
  classify_grid(g);
  return g;
}

// ---- transits --------------------------------------------------------------------
std::array<double, 6> neighbor_weights(const DielectricGrid& grid, const Vec3i& node) {
  const int n = grid.n;
  for (int a = 0; a < 3; ++a)
    if (node[a] < 0 || node[a] >= n)
      throw std::invalid_argument("neighbor_weights: node outside lattice");
  if (grid.conductor(node.x, node.y, node.z) >= 0)
    throw std::invalid_argument("neighbor_weights: node is a conductor voxel");
  const double ev = grid.eps_at(node.x, node.y, node.z);
  std::array<double, 6> beta;
  double sum = 0;
  for (int d = 0; d < 6; ++d) {
    Vec3i nb = node;
    const int a = kDirAxis[d];
    nb[a] += kDirSign[d];
    double alpha = 1.0;
    if (nb[a] >= 0 && nb[a] < n && grid.conductor(nb.x, nb.y, nb.z) < 0) {
      const double en = grid.eps_at(nb.x, nb.y, nb.z);
      alpha = en / (en + ev);
    }
    beta[d] = alpha;
    sum += alpha;
  }
  for (double& b : beta) b /= sum;
  return beta;
}

std::vector<Exit> microwalk_transits(const DielectricGrid& grid, std::vector<SplitMix64>& rngs,
                                     int step_cap, int device) {
  frw_ctx* ctx = Device::get(device).ctx();
  ensure_grid(ctx, grid);
  const int64_t count = static_cast<int64_t>(rngs.size());
  std::vector<uint64_t> st(count);
  for (int64_t t = 0; t < count; ++t) st[t] = rngs[t].state();
  std::vector<int32_t> panel(count), steps(count), cond(count);
  std::vector<int64_t> nd(count);
  frw_mw_params p{FRW_RNG_SPLITMIX_STATES, 0, 0, count, step_cap, 0, st.data()};
  frw_mw_out o{};
  o.panels = panel.data();
  o.steps = steps.data();
  o.cond = cond.data();
  o.exit_nd = nd.data();
  throw_status(ctx, frw_microwalk_batch(ctx, &p, &o));
  std::vector<Exit> out(count);
  for (int64_t t = 0; t < count; ++t) {
    out[t] = exit_from_grid(grid, panel[t], steps[t], cond[t], nd[t]);
    rngs[t].skip(static_cast<uint64_t>(steps[t]));
  }
  return out;
}

Exit microwalk_transit(const DielectricGrid& grid, SplitMix64& rng, MicroWalkScratch& scratch,
                       int step_cap) {
  scratch.prepare(grid.n);
  std::vector<SplitMix64> r{rng};
  const Exit e = microwalk_transits(grid, r, step_cap, scratch.device)[0];
  rng = r[0];
  return e;
}

Exit microwalk_transit(const DielectricGrid& grid, SplitMix64& rng) {
  MicroWalkScratch scratch;
  return microwalk_transit(grid, rng, scratch, 0);
}

void upload_structure(frw_ctx* ctx, const Structure& s) {
  std::vector<int32_t> ids;
  std::vector<double> cb, db, de;
  for (const auto& c : s.conductors) {
    ids.push_back(c.id);
    for (int a = 0; a < 3; ++a) cb.push_back(c.box.lo[a]);
    for (int a = 0; a < 3; ++a) cb.push_back(c.box.hi[a]);
  }
  for (const auto& d : s.dielectrics) {
    for (int a = 0; a < 3; ++a) db.push_back(d.box.lo[a]);
    for (int a = 0; a < 3; ++a) db.push_back(d.box.hi[a]);
    de.push_back(d.eps_r);
  }
  frw_structure fs{};
  fs.n_cond = static_cast<int32_t>(ids.size());
  fs.cond_id = ids.data();
  fs.cond_box = cb.data();
  fs.n_diel = static_cast<int32_t>(de.size());
  fs.diel_box = db.data();
  fs.diel_eps = de.data();
  fs.background_eps = s.background_eps;
  for (int a = 0; a < 3; ++a) {
    fs.world[a] = s.world.lo[a];
    fs.world[3 + a] = s.world.hi[a];
  }
  uint64_t h = 0xcbf29ce484222325ull;
  h = fnv(h, ids.data(), 4 * ids.size());
  h = fnv(h, cb.data(), 8 * cb.size());
  h = fnv(h, db.data(), 8 * db.size());
  h = fnv(h, de.data(), 8 * de.size());
  h = fnv(h, &fs.background_eps, 8);
  h = fnv(h, fs.world, sizeof fs.world);
  h |= 1;
  std::lock_guard<std::mutex> lk(g_mu);
  if (structure_fp()[ctx] == h) return;
  throw_status(ctx, frw_upload_structure(ctx, &fs));
  structure_fp()[ctx] = h;
}

std::vector<Exit> microwalk_structure_transits(const Structure& s, const std::vector<Cube>& cubes,
                                               int n, bool with_conductors,
                                               std::vector<SplitMix64>& rngs, int step_cap,
                                               int device) {
  if (cubes.size() != rngs.size())
    throw std::invalid_argument("microwalk_structure_transits: one rng per cube");
  frw_ctx* ctx = Device::get(device).ctx();
  upload_structure(ctx, s);
  const int count = static_cast<int>(cubes.size());
  std::vector<double> cb(4 * cubes.size());
  std::vector<uint64_t> st(count);
  for (int t = 0; t < count; ++t) {
    cb[4 * t] = cubes[t].center.x;
    cb[4 * t + 1] = cubes[t].center.y;
    cb[4 * t + 2] = cubes[t].center.z;
    cb[4 * t + 3] = cubes[t].half_width;
    st[t] = rngs[t].state();
  }
  std::vector<frw_exit> ex(count);
  throw_status(ctx, frw_structure_transits(ctx, n, count, cb.data(), with_conductors ? 1 : 0,
                                           st.data(), step_cap, ex.data()));
  std::vector<Exit> out(count);
  for (int t = 0; t < count; ++t) {
    const frw_exit& x = ex[t];
    Exit& e = out[t];
    if (x.kind < 0) {  // EngulfedStart: no draw consumed
      e.kind = Exit::Kind::Conductor;
      e.conductor_id = -1;
      e.steps = 0;
      continue;
    }
    e.kind = x.kind == 0 ? Exit::Kind::Surface : Exit::Kind::Conductor;
    e.panel = x.panel;
    e.conductor_id = x.kind == 1 ? s.conductors.at(x.conductor).id : -1;
    e.point = {x.point[0], x.point[1], x.point[2]};
    e.voxel = {x.voxel[0], x.voxel[1], x.voxel[2]};
    e.dir = x.dir;
    e.steps = x.steps;
    rngs[t].skip(static_cast<uint64_t>(x.steps));
  }
  return out;
}

Exit microwalk_transit_lazy(const Structure& s, const Cube& cube, int n, SplitMix64& rng,
                            MicroWalkScratch& scratch, int step_cap) {
  scratch.prepare(n);
  std::vector<SplitMix64> r{rng};
  const Exit e = microwalk_structure_transits(s, {cube}, n, false, r, step_cap, scratch.device)[0];
  rng = r[0];
  return e;
}

Exit microwalk_e_transit(const Structure& s, const Vec3& center, double base_half_width,
                         double expansion, int n, SplitMix64& rng, MicroWalkScratch& scratch,
                         int step_cap) {
  if (expansion < 1.0) throw std::invalid_argument("microwalk_e_transit: expansion must be >= 1");
  const double wall = s.world.chebyshev_to_wall(center);
  const double half = std::min(expansion * base_half_width, wall);
  if (!(half > 0))
    throw std::invalid_argument("microwalk_e_transit: center is on or outside the world wall");
  scratch.prepare(n);
  std::vector<SplitMix64> r{rng};
  const Exit e = microwalk_structure_transits(s, {transit_cube(center, half, n)}, n, true, r,
                                              step_cap, scratch.device)[0];
  if (e.kind == Exit::Kind::Conductor && e.conductor_id < 0)
    throw EngulfedStart("transit start voxel lies inside a conductor");
  rng = r[0];
  return e;
}

Exit microwalk_e_transit(const Structure& s, const Vec3& center, double base_half_width,
                         double expansion, int n, SplitMix64& rng) {
  MicroWalkScratch scratch;
  return microwalk_e_transit(s, center, base_half_width, expansion, n, rng, scratch, 0);
}

TransitBatch microwalk_transit_batch(int n, const std::vector<double>& eps, const Vec3& c,
                                     double half_width, uint64_t seed, uint64_t stream_begin,
                                     int64_t count, RngMode rng, bool per_transit, int device) {
  frw_ctx* ctx = Device::get(device).ctx();
  DielectricGrid g;
  g.n = n;
  g.cube = {c, half_width};
  g.eps = eps;
  ensure_grid(ctx, g);
  TransitBatch out;
  out.hist.assign(6ull * n * n, 0);
  if (per_transit) {
    out.panels.resize(count);
    out.steps.resize(count);
  }
  frw_mw_params p{rng == RngMode::Philox ? FRW_RNG_PHILOX : FRW_RNG_SPLITMIX_PARITY,
                  seed, stream_begin, count, 0, 0, nullptr};
  frw_mw_out o{};
  o.hist = out.hist.data();
  o.step_sum = &out.step_sum;
  o.step_sumsq = &out.step_sumsq;
  if (per_transit) {
    o.panels = out.panels.data();
    o.steps = out.steps.data();
  }
  throw_status(ctx, frw_microwalk_batch(ctx, &p, &o));
  return out;
}

ReferenceSolution reference_capacitance(const Structure& s, int resolution, int device) {
  frw_ctx* ctx = Device::get(device).ctx();
  std::vector<int32_t> ids;
  std::vector<double> cb, db, de;
  for (const auto& c : s.conductors) {
    ids.push_back(c.id);
    for (int a = 0; a < 3; ++a) cb.push_back(c.box.lo[a]);
    for (int a = 0; a < 3; ++a) cb.push_back(c.box.hi[a]);
  }
  for (const auto& d : s.dielectrics) {
    for (int a = 0; a < 3; ++a) db.push_back(d.box.lo[a]);
    for (int a = 0; a < 3; ++a) db.push_back(d.box.hi[a]);
    de.push_back(d.eps_r);
  }
  frw_structure fs{};
  fs.n_cond = static_cast<int32_t>(ids.size());
  fs.cond_id = ids.data();
  fs.cond_box = cb.data();
  fs.n_diel = static_cast<int32_t>(de.size());
  fs.diel_box = db.data();
  fs.diel_eps = de.data();
  fs.background_eps = s.background_eps;
  for (int a = 0; a < 3; ++a) {
    fs.world[a] = s.world.lo[a];
    fs.world[3 + a] = s.world.hi[a];
  }
  ReferenceSolution r;
  r.resolution = resolution;
  r.terminal_ids.assign(ids.begin(), ids.end());
  r.capacitance.assign(ids.size() * ids.size(), 0.0);
  throw_status(ctx, frw_reference_capacitance(ctx, &fs, resolution, r.capacitance.data(),
                                              &r.residual));
  return r;
}

DiscreteSGF solve_sgf(const DielectricGrid& g, bool with_kernels, int device) {
  if (g.has_mask()) return direct_sgf(g, with_kernels).sgf;  // conductor voxels: host direct
  frw_ctx* ctx = Device::get(device).ctx();
  const size_t P = 6ull * g.n * g.n;
  DiscreteSGF out;
  out.n = g.n;
  out.pitch = g.pitch();
  out.probs.resize(P);
  std::vector<double> ker(with_kernels ? 3 * P : 0);
  DielectricGrid cls;  // the grid's own classification (callers may not have run it)
  cls.n = g.n;
  cls.cube = g.cube;
  cls.eps = g.eps;
  classify_grid(cls);
  bool exact = cls.tag != GridTag::General;  // (classify_grid compares at rel-tol 1e-9)
  if (exact) {
    const int ax = cls.tag == GridTag::Stratified ? cls.strat_axis : 0;
    for (int k = 0; k < g.n && exact; ++k)
      for (int j = 0; j < g.n && exact; ++j)
        for (int i = 0; i < g.n && exact; ++i) {
          const int t = ax == 0 ? i : (ax == 1 ? j : k);
          exact = g.eps_at(i, j, k) ==
                  g.eps_at(ax == 0 ? t : 0, ax == 1 ? t : 0, ax == 2 ? t : 0);
        }
  }
  if (exact) {
    // a stratified (or uniform) grid is the separable system the stratified
    // cache solves: the same exact direct solver (frw_sgf_solve), so a
    // cached key and the solve of its canonical grid agree bit for bit;
    // its unit-pitch kernels scale with 1 / pitch
    const int axis = cls.tag == GridTag::Stratified ? cls.strat_axis : 0;
    std::vector<double> layers(g.n);
    for (int t = 0; t < g.n; ++t)
      layers[t] = g.eps_at(axis == 0 ? t : 0, axis == 1 ? t : 0, axis == 2 ? t : 0);
    throw_status(ctx, frw_sgf_solve(ctx, g.n, 1, &axis, layers.data(), out.probs.data(),
                                    with_kernels ? ker.data() : nullptr));
    if (with_kernels && out.pitch != 1.0)
      for (double& k : ker) k /= out.pitch;
  } else {
    const int rc = frw_grid_sgf_solve(ctx, g.n, 1, g.eps.data(), g.cube.half_width,
                                      out.probs.data(), with_kernels ? ker.data() : nullptr,
                                      nullptr);
    // the PCG stalled: the direct factorisation, as the reference falls back
    // to SimplicialLDLT (sgf.cpp:170-176)
    if (rc == FRW_ESOLVE && g.n <= 32) return direct_sgf(g, with_kernels).sgf;
    throw_status(ctx, rc);
  }
  out.cdf.resize(P);
  double run = 0;
  for (size_t b = 0; b < P; ++b) out.cdf[b] = run += out.probs[b];
  if (with_kernels)
    for (int a = 0; a < 3; ++a) out.grad_kernels[a].assign(ker.begin() + a * P, ker.begin() + (a + 1) * P);
  return out;
}

FDSystem assemble_system(const DielectricGrid& g) {
  if (g.n < 1 || g.eps.size() != static_cast<size_t>(g.n) * g.n * g.n)
    throw std::invalid_argument("assemble_system: malformed grid");
  FDSystem s;
  s.grid = g;
  s.n = g.n;
  return s;
}

DiscreteSGF solve_sgf(const FDSystem& sys, bool with_kernels) {
  return solve_sgf(sys.grid, with_kernels);
}

double expected_steps(const FDSystem& sys) { return expected_steps(sys.grid); }

DistributionReport compare_distribution(const std::vector<double>& exact,
                                        const std::function<int(SplitMix64&)>& sampler,
                                        long n_samples, SplitMix64& rng) {
  if (n_samples < 10000) throw std::invalid_argument("compare_distribution: too few samples");
  DistributionReport r;
  r.exact = exact;
  r.samples = n_samples;
  std::vector<long> hist(exact.size(), 0);
  for (long i = 0; i < n_samples; ++i) ++hist.at(static_cast<size_t>(sampler(rng)));
  r.empirical.resize(exact.size());
  for (size_t b = 0; b < exact.size(); ++b) {
    r.empirical[b] = static_cast<double>(hist[b]) / n_samples;
    r.tv_distance += std::fabs(r.empirical[b] - exact[b]);
  }
  r.tv_distance *= 0.5;
  // consecutive bins pooled to an expected count >= 5; the tail joins the
  // last group (or forms one when there is none)
  std::vector<double> obs, expct;
  double o = 0, e = 0;
  for (size_t b = 0; b < exact.size(); ++b) {
    e += exact[b] * n_samples;
    o += static_cast<double>(hist[b]);
    if (e >= 5.0) {
      obs.push_back(o);
      expct.push_back(e);
      o = e = 0;
    }
  }
  if (o > 0 || e > 0) {
    if (obs.empty()) {
      obs.push_back(o);
      expct.push_back(std::max(e, 1e-12));
    } else {
      obs.back() += o;
      expct.back() += e;
    }
  }
  for (size_t k = 0; k < obs.size(); ++k)
    r.gof_statistic += (obs[k] - expct[k]) * (obs[k] - expct[k]) / expct[k];
  r.pooled_bins = static_cast<int>(obs.size());
  // Wilson-Hilferty: chi2_{1-p}(d) ~ d (1 - 2/(9d) + z sqrt(2/(9d)))^3, z = 3.0902
  const double d = std::max(r.pooled_bins - 1, 1);
  const double w = 1.0 - 2.0 / (9.0 * d) + 3.090232306167813 * std::sqrt(2.0 / (9.0 * d));
  r.gof_critical = d * w * w * w;
  return r;
}

double expected_steps(const DielectricGrid& g, int device) {
  if (g.has_mask()) return direct_sgf(g, false).expected_steps;
  frw_ctx* ctx = Device::get(device).ctx();
  double st = 0;
  const int rc = frw_grid_sgf_solve(ctx, g.n, 1, g.eps.data(), g.cube.half_width, nullptr,
                                    nullptr, &st);
  if (rc == FRW_ESOLVE && g.n <= 32) return direct_sgf(g, false).expected_steps;
  throw_status(ctx, rc);
  return st;
}

namespace {
double exp_eps(SplitMix64& rng) {  // oracle.cpp:300-303
  return std::max(-10.0 * std::log1p(-rng.uniform()), 1e-9);
}
DielectricGrid blank_grid(int n) {  // oracle.cpp:305-311
  DielectricGrid g;
  g.n = n;
  g.cube = {{0, 0, 0}, n / 2.0};
  g.eps.assign(static_cast<size_t>(n) * n * n, 1.0);
  return g;
}
}  // namespace

DielectricGrid random_voxel_grid(int n, SplitMix64& rng) {
  DielectricGrid g = blank_grid(n);
  for (auto& e : g.eps) e = exp_eps(rng);
  classify_grid(g);
  return g;
}

DielectricGrid random_block_grid(int n, int blocks, SplitMix64& rng) {
  DielectricGrid g = blank_grid(n);
  for (int b = 0; b < blocks; ++b) {
    int lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
      const int x = static_cast<int>(rng.uniform() * n);
      const int y = static_cast<int>(rng.uniform() * n);
      lo[a] = std::min(std::min(x, y), n - 1);
      hi[a] = std::min(std::max(x, y), n - 1);
    }
    const double e = exp_eps(rng);
    for (int k = lo[2]; k <= hi[2]; ++k)
      for (int j = lo[1]; j <= hi[1]; ++j)
        for (int i = lo[0]; i <= hi[0]; ++i) g.eps[g.index(i, j, k)] = e;
  }
  classify_grid(g);
  return g;
}

}  // namespace frwcap
