// sgf.cpp -- stratified-SGF miss solver and cache of the B200 build.
//
// The walk-time lookup and CDF sampling run on the device (walk.cu); this
// file solves the canonical grid of a missing key on the host and keeps
// the host copy of the table.  Algorithm restated from the reference:
//   FD system       proj/src/sgf.cpp:57-155 (alpha = e_i/(e_i+e_v), absorbing
//                   faces alpha = 1, bit-symmetric s_ii = diag(eps) A_II)
//   adjoint solve   sgf.cpp:162-290 (s_ii z = b, y = eps .* z, probs = A_IB^T y;
//                   Jacobi-PCG at rel. tol 1e-10, cap 20*rows)
//   kernels         sgf.cpp:265-288 (central differences about the start node)
//   expected_steps  sgf.cpp:292-299
//   keys / cache    sgf_cache.cpp:13-153, SGF1 files sgf_cache.cpp:210-324
// The solve is matrix-free on the 7-point stencil.  There is no direct
// (LDLT) fallback: a non-converging PCG raises SolveError.
#include <algorithm>
#include <atomic>
#include <bit>
#include <cmath>
#include <cstring>
#include <fstream>
#include <thread>

#include "frwcap.hpp"

namespace frwcap {

double round_sig(double x, int digits) {
  if (x == 0 || !std::isfinite(x)) return x;
  const double e10 = std::floor(std::log10(std::fabs(x)));
  const double mag = std::pow(10.0, digits - 1 - e10);
  return std::round(x * mag) / mag;
}

namespace {
uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
}  // namespace

size_t ProfileKeyHash::operator()(const ProfileKey& k) const {
  uint64_t h = mix64((static_cast<uint64_t>(k.n) << 8) ^ static_cast<uint64_t>(k.axis));
  for (double v : k.layers) h = mix64(h ^ std::bit_cast<uint64_t>(v));
  return static_cast<size_t>(h);
}

ProfileKey profile_key(int n, int axis, const std::vector<double>& layers) {
  if (static_cast<int>(layers.size()) != n)
    throw std::invalid_argument("profile_key: expected one layer per slice");
  if (axis < 0 || axis > 2) throw std::invalid_argument("profile_key: axis out of range");
  ProfileKey k;
  k.n = n;
  k.axis = axis;
  for (double v : layers) k.layers.push_back(round_sig(v, 6));
  bool uniform = true;
  for (double v : k.layers) uniform = uniform && v == k.layers[0];
  if (uniform) k.axis = 0;
  return k;
}

namespace {

// matrix-free s_ii of an unmasked n^3 lattice
struct Stencil {
  int n = 0;
  size_t m = 0;
  std::vector<double> eps, diag, rowsum;
  std::vector<std::array<double, 6>> off;  // 0 where the face absorbs

  Stencil(int n_, const std::vector<double>& e) : n(n_), m(size_t(n_) * n_ * n_), eps(e) {
    diag.resize(m);
    rowsum.resize(m);
    off.resize(m);
    for (int k = 0; k < n; ++k)
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
          const size_t v = (size_t(k) * n + j) * n + i;
          const double ev = eps[v];
          double rs = 0;
          const int c[3] = {i, j, k};
          for (int d = 0; d < 6; ++d) {
            const int a = d >> 1, s = (d & 1) ? 1 : -1;
            int nb[3] = {c[0], c[1], c[2]};
            nb[a] += s;
            off[v][d] = 0;
            if (nb[a] < 0 || nb[a] >= n) {
              rs += 1.0;
              continue;
            }
            const double ei = eps[(size_t(nb[2]) * n + nb[1]) * n + nb[0]];
            off[v][d] = -(ev * ei) / (ev + ei);
            rs += ei / (ei + ev);
          }
          rowsum[v] = rs;
          diag[v] = ev * rs;
        }
  }

  void apply(const std::vector<double>& x, std::vector<double>& y) const {
    const long st[6] = {-1, 1, -long(n), long(n), -long(n) * n, long(n) * n};
    for (size_t v = 0; v < m; ++v) {
      double acc = diag[v] * x[v];
      for (int d = 0; d < 6; ++d)
        if (off[v][d] != 0.0) acc += off[v][d] * x[v + st[d]];
      y[v] = acc;
    }
  }

  // Jacobi-PCG from zero; converged when |r|^2 < tol^2 |b|^2
  std::vector<double> solve(const std::vector<double>& b, double tol = 1e-10) const {
    std::vector<double> x(m, 0.0), r = b, z(m), p(m), t(m);
    auto dot = [&](const std::vector<double>& a, const std::vector<double>& c) {
      double s = 0;
      for (size_t i = 0; i < m; ++i) s += a[i] * c[i];
      return s;
    };
    const double b2 = dot(b, b);
    if (b2 == 0) return x;
    const double thr = tol * tol * b2;
    if (dot(r, r) < thr) return x;
    for (size_t i = 0; i < m; ++i) p[i] = r[i] / diag[i];
    double rz = dot(r, p);
    const size_t cap = 20 * m;
    for (size_t it = 0; it < cap; ++it) {
      apply(p, t);
      const double a = rz / dot(p, t);
      for (size_t i = 0; i < m; ++i) {
        x[i] += a * p[i];
        r[i] -= a * t[i];
      }
      const double rr = dot(r, r);
      if (rr < thr) return x;
      for (size_t i = 0; i < m; ++i) z[i] = r[i] / diag[i];
      const double old = rz;
      rz = dot(r, z);
      const double beta = rz / old;
      for (size_t i = 0; i < m; ++i) p[i] = z[i] + beta * p[i];
    }
    throw SolveError("transition cube solve failed: PCG did not converge",
                     std::sqrt(dot(r, r) / b2));
  }

  // A_IB^T (eps .* z): the boundary row of the adjoint solution
  std::vector<double> boundary(const std::vector<double>& z) const {
    std::vector<double> out(6 * size_t(n) * n, 0.0);
    for (int k = 0; k < n; ++k)
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
          const size_t v = (size_t(k) * n + j) * n + i;
          const int c[3] = {i, j, k};
          for (int d = 0; d < 6; ++d) {
            const int a = d >> 1;
            const int nb = c[a] + ((d & 1) ? 1 : -1);
            if (nb >= 0 && nb < n) continue;
            const int u = a == 0 ? j : i;
            const int w = a == 2 ? j : k;
            out[(size_t(d) * n + w) * n + u] = eps[v] * z[v];
          }
        }
    return out;
  }
};

DiscreteSGF solve_stencil(const Stencil& S, double half_width, bool with_kernels) {
  const int n = S.n;
  DiscreteSGF out;
  out.n = n;
  out.pitch = 2.0 * half_width / n;
  const int c = (n - 1) / 2;
  const size_t crow = (size_t(c) * n + c) * n + c;
  std::vector<double> e(S.m, 0.0);
  e[crow] = 1.0;
  const std::vector<double> p = S.boundary(S.solve(e));
  double total = 0, lowest = 0;
  for (double v : p) {
    total += v;
    lowest = std::min(lowest, v);
  }
  if (std::fabs(total - 1.0) > 1e-9 || lowest < -1e-9)
    throw SolveError("transition cube solve failed normalization check", std::fabs(total - 1));
  out.probs.resize(p.size());
  out.cdf.resize(p.size());
  double run = 0;
  for (size_t b = 0; b < p.size(); ++b) {
    out.probs[b] = std::max(p[b], 0.0);
    run += out.probs[b];
    out.cdf[b] = run;
  }
  if (!with_kernels) return out;
  for (int a = 0; a < 3; ++a) {
    out.grad_kernels[a].assign(p.size(), 0.0);
    int up[3] = {c, c, c}, dn[3] = {c, c, c};
    up[a] += 1;
    dn[a] -= 1;
    const bool hu = up[a] < n, hd = dn[a] >= 0;
    std::vector<double> rhs(S.m, 0.0);
    double denom;
    auto idx = [&](const int* q) { return (size_t(q[2]) * n + q[1]) * n + q[0]; };
    if (hu && hd) {
      rhs[idx(up)] += 1.0;
      rhs[idx(dn)] -= 1.0;
      denom = 2.0 * out.pitch;
    } else if (hu) {
      rhs[idx(up)] += 1.0;
      rhs[crow] -= 1.0;
      denom = out.pitch;
    } else if (hd) {
      rhs[crow] += 1.0;
      rhs[idx(dn)] -= 1.0;
      denom = out.pitch;
    } else {
      continue;  // n = 1: zero kernel
    }
    const std::vector<double> k = S.boundary(S.solve(rhs));
    for (size_t b = 0; b < k.size(); ++b) out.grad_kernels[a][b] = k[b] / denom;
  }
  return out;
}

}  // namespace

DiscreteSGF solve_canonical(const ProfileKey& key, bool with_kernels) {
  const int n = key.n;
  if (static_cast<int>(key.layers.size()) != n)
    throw std::invalid_argument("canonical_grid: malformed key");
  std::vector<double> eps(size_t(n) * n * n);
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        const int v[3] = {i, j, k};
        eps[(size_t(k) * n + j) * n + i] = key.layers[v[key.axis]];
      }
  // canonical unit-pitch cube: half width n/2 (sgf_cache.cpp:78-96)
  return solve_stencil(Stencil(n, eps), n / 2.0, with_kernels);
}


// ---- cache -------------------------------------------------------------------

std::shared_ptr<const DiscreteSGF> StratifiedSgfCache::find(const ProfileKey& key) const {
  std::lock_guard<std::mutex> lk(mu_);
  auto it = map_.find(key);
  return it == map_.end() ? nullptr : it->second;
}

std::shared_ptr<const DiscreteSGF> StratifiedSgfCache::get(const ProfileKey& key) {
  {
    std::lock_guard<std::mutex> lk(mu_);
    auto it = map_.find(key);
    if (it != map_.end()) {
      ++hits_;
      return it->second;
    }
    ++misses_;
  }
  auto sgf = std::make_shared<DiscreteSGF>(solve_canonical(key, true));
  std::lock_guard<std::mutex> lk(mu_);
  auto [it, inserted] = map_.emplace(key, sgf);  // first stored result wins
  if (inserted && capacity_ > 0 && map_.size() > capacity_) map_.erase(map_.begin());
  return it->second;
}

void StratifiedSgfCache::solve_many(const std::vector<ProfileKey>& keys, int threads) {
  std::vector<ProfileKey> todo;
  {
    std::lock_guard<std::mutex> lk(mu_);
    for (const auto& k : keys)
      if (!map_.count(k)) todo.push_back(k);
    misses_ += todo.size();
  }
  if (todo.empty()) return;
  if (threads <= 0) threads = std::max(1u, std::thread::hardware_concurrency());
  threads = std::min<int>(threads, static_cast<int>(todo.size()));
  std::atomic<size_t> next{0};
  std::vector<std::exception_ptr> errs(threads);
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      try {
        for (size_t i = next++; i < todo.size(); i = next++) {
          auto sgf = std::make_shared<DiscreteSGF>(solve_canonical(todo[i], true));
          std::lock_guard<std::mutex> lk(mu_);
          map_.emplace(todo[i], sgf);
        }
      } catch (...) {
        errs[t] = std::current_exception();
      }
    });
  for (auto& th : pool) th.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

std::shared_ptr<const DiscreteSGF> StratifiedSgfCache::insert(
    const ProfileKey& key, std::shared_ptr<const DiscreteSGF> sgf) {
  std::lock_guard<std::mutex> lk(mu_);
  return map_.emplace(key, std::move(sgf)).first->second;
}

void StratifiedSgfCache::count_misses(uint64_t k) {
  std::lock_guard<std::mutex> lk(mu_);
  misses_ += k;
}

StratifiedSgfCache::Stats StratifiedSgfCache::stats() const {
  std::lock_guard<std::mutex> lk(mu_);
  return {hits_, misses_, map_.size()};
}

void StratifiedSgfCache::clear() {
  std::lock_guard<std::mutex> lk(mu_);
  map_.clear();
}

std::vector<std::pair<ProfileKey, std::shared_ptr<const DiscreteSGF>>>
StratifiedSgfCache::entries() const {
  std::lock_guard<std::mutex> lk(mu_);
  return {map_.begin(), map_.end()};
}

namespace {
void put_u32(std::string& o, uint32_t v) {
  for (int i = 0; i < 4; ++i) o.push_back(static_cast<char>(v >> (8 * i)));
}
void put_u64(std::string& o, uint64_t v) {
  for (int i = 0; i < 8; ++i) o.push_back(static_cast<char>(v >> (8 * i)));
}
void put_f64(std::string& o, double v) { put_u64(o, std::bit_cast<uint64_t>(v)); }

struct In {
  const std::string& b;
  size_t pos = 0;
  void need(size_t k) const {
    if (pos + k > b.size()) throw std::runtime_error("SGF cache file is truncated");
  }
  uint64_t uint(int bytes) {
    need(bytes);
    uint64_t v = 0;
    for (int i = 0; i < bytes; ++i)
      v |= static_cast<uint64_t>(static_cast<unsigned char>(b[pos++])) << (8 * i);
    return v;
  }
  double f64() { return std::bit_cast<double>(uint(8)); }
};
}  // namespace

// SGF1 layout (sgf_cache.cpp:210-247): "SGF1", u32 n, u64 count, then per
// entry u32 axis, u8 expanded, u8 has_sig, u64 sig, u32 nlayers, f64 layers,
// f64 pitch, u64 nprobs, f64 probs, u8 has_kernels, f64 kernels[3][nprobs]
void StratifiedSgfCache::save(const std::string& path, int only_n) const {
  const auto all = entries();
  int n = only_n;
  size_t count = 0;
  for (const auto& [k, v] : all) {
    if (only_n > 0 && k.n != only_n) continue;
    if (n == 0) n = k.n;
    if (k.n != n)
      throw std::invalid_argument("SGF cache files hold a single lattice size; clear between sizes");
    ++count;
  }
  std::string o = "SGF1";
  put_u32(o, static_cast<uint32_t>(n));
  put_u64(o, count);
  for (const auto& [k, v] : all) {
    if (only_n > 0 && k.n != only_n) continue;
    put_u32(o, static_cast<uint32_t>(k.axis));
    o.push_back(0);
    o.push_back(0);
    put_u64(o, 0);
    put_u32(o, static_cast<uint32_t>(k.layers.size()));
    for (double x : k.layers) put_f64(o, x);
    put_f64(o, v->pitch);
    put_u64(o, v->probs.size());
    for (double x : v->probs) put_f64(o, x);
    const bool kern = !v->grad_kernels[0].empty();
    o.push_back(kern ? 1 : 0);
    if (kern)
      for (const auto& g : v->grad_kernels)
        for (double x : g) put_f64(o, x);
  }
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) throw std::runtime_error("cannot open " + path + " for writing");
  f.write(o.data(), static_cast<std::streamsize>(o.size()));
  if (!f) throw std::runtime_error("short write to " + path);
}

size_t StratifiedSgfCache::load(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot open " + path);
  const std::string buf((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  In r{buf};
  r.need(4);
  if (buf.compare(0, 4, "SGF1") != 0) throw std::runtime_error(path + " is not an SGF cache file");
  r.pos = 4;
  const int n = static_cast<int>(r.uint(4));
  if (n < 1 || n > 4096) throw std::runtime_error("SGF cache: bad lattice size");
  const uint64_t count = r.uint(8);
  const uint64_t panels = 6ull * n * n;
  size_t loaded = 0;
  for (uint64_t e = 0; e < count; ++e) {
    ProfileKey key;
    key.n = n;
    key.axis = static_cast<int>(r.uint(4));
    if (key.axis < 0 || key.axis > 2) throw std::runtime_error("SGF cache: bad axis");
    const bool expanded = r.uint(1) != 0;
    const bool has_sig = r.uint(1) != 0;
    r.uint(8);
    if (static_cast<int>(r.uint(4)) != n) throw std::runtime_error("SGF cache: layer count mismatch");
    key.layers.resize(n);
    for (double& v : key.layers) v = r.f64();
    auto sgf = std::make_shared<DiscreteSGF>();
    sgf->n = n;
    sgf->pitch = r.f64();
    if (!(sgf->pitch > 0)) throw std::runtime_error("SGF cache: bad pitch");
    if (r.uint(8) != panels) throw std::runtime_error("SGF cache: bad panel count");
    sgf->probs.resize(panels);
    double sum = 0, lo = 0;
    for (double& v : sgf->probs) {
      v = r.f64();
      sum += v;
      lo = std::min(lo, v);
    }
    if (std::fabs(sum - 1.0) > 1e-9 || lo < -1e-9)
      throw std::runtime_error("SGF cache: entry fails normalization");
    sgf->cdf.resize(panels);
    double acc = 0;
    for (uint64_t i = 0; i < panels; ++i) sgf->cdf[i] = acc += sgf->probs[i];
    if (r.uint(1) != 0)
      for (auto& g : sgf->grad_kernels) {
        g.resize(panels);
        double ks = 0;
        for (double& v : g) ks += v = r.f64();
        if (std::fabs(ks) > 1e-9) throw std::runtime_error("SGF cache: kernel fails zero-sum check");
      }
    // expanded / conductor-signature keys belong to the MicroWalk-E cache,
    // which this build does not serve from the table; keep them out
    if (!expanded && !has_sig) {
      std::lock_guard<std::mutex> lk(mu_);
      map_.emplace(std::move(key), std::move(sgf));
      ++loaded;
    }
  }
  if (r.pos != buf.size()) throw std::runtime_error("SGF cache: trailing bytes");
  return loaded;
}

}  // namespace frwcap
