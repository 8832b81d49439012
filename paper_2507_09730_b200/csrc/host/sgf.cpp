// sgf.cpp -- stratified-SGF cache of the B200 build.
//
// The walk-time lookup and CDF sampling run on the device (walk.cu); so do
// the canonical solves of missing keys (frw_sgf_solve, sgf_solve.cu).  This
// file keeps the host copy of the table (keys, SGF1 files).  The solver
// restates the reference:
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
  uint64_t h = mix64((static_cast<uint64_t>(k.n) << 8) ^ static_cast<uint64_t>(k.axis) ^
                     (static_cast<uint64_t>(k.expanded) << 40));
  for (double v : k.layers) h = mix64(h ^ std::bit_cast<uint64_t>(v));
  if (k.conductor_sig) h = mix64(h ^ *k.conductor_sig ^ 0x5bd1e995ull);
  return static_cast<size_t>(h);
}

ProfileKey profile_key(int n, int axis, const std::vector<double>& layers, bool expanded,
                       std::optional<uint64_t> conductor_sig) {
  if (static_cast<int>(layers.size()) != n)
    throw std::invalid_argument("profile_key: expected one layer per slice");
  if (axis < 0 || axis > 2) throw std::invalid_argument("profile_key: axis out of range");
  ProfileKey k;
  k.n = n;
  k.axis = axis;
  for (double v : layers) k.layers.push_back(round_sig(v, 6));
  bool uniform = true;
  for (double v : k.layers) uniform = uniform && v == k.layers[0];
  if (uniform) k.axis = 0;  // sgf_cache.cpp:40-42
  k.expanded = expanded;
  k.conductor_sig = conductor_sig;
  return k;
}

ProfileKey profile_key(const StratifiedProfile& profile, int n) {
  return profile_key(n, profile.axis, profile.layers);
}

ProfileKey profile_key(const DielectricGrid& grid) {
  if (grid.tag == GridTag::General)
    throw std::invalid_argument("profile_key: grid is not stratified");
  const int axis = grid.tag == GridTag::Stratified ? grid.strat_axis : 0;
  std::vector<double> layers(grid.n);
  for (int t = 0; t < grid.n; ++t)  // the layer along the axis, at (0, 0) across
    layers[t] = grid.eps_at(axis == 0 ? t : 0, axis == 1 ? t : 0, axis == 2 ? t : 0);
  return profile_key(grid.n, axis, layers);
}

uint64_t conductor_signature(const DielectricGrid& grid) {
  uint64_t h = mix64(static_cast<uint64_t>(grid.n));
  if (!grid.has_mask()) return h;
  for (size_t i = 0; i < grid.conductor_mask.size(); ++i)
    if (grid.conductor_mask[i] >= 0)
      h = mix64(h ^ (static_cast<uint64_t>(i) << 32 ^
                     static_cast<uint32_t>(grid.conductor_mask[i])));
  return h;
}


// canonical unit-pitch solves of stratified keys (sgf_cache.cpp:78-131) on the
// device solver (frw_sgf_solve, sgf_solve.cu)
namespace {
std::vector<std::shared_ptr<DiscreteSGF>> solve_keys(const std::vector<ProfileKey>& keys,
                                                     bool with_kernels, int device) {
  std::vector<std::shared_ptr<DiscreteSGF>> out;
  if (keys.empty()) return out;
  const int n = keys[0].n;
  std::vector<int> axes;
  std::vector<double> layers;
  for (const auto& k : keys) {
    if (k.n != n || static_cast<int>(k.layers.size()) != n)
      throw std::invalid_argument("canonical_grid: malformed key");
    axes.push_back(k.axis);
    layers.insert(layers.end(), k.layers.begin(), k.layers.end());
  }
  const size_t P = 6ull * n * n;
  std::vector<double> pr(P * keys.size()), ke(with_kernels ? 3 * P * keys.size() : 0);
  frw_ctx* ctx = Device::get(device).ctx();
  const int rc = frw_sgf_solve(ctx, n, static_cast<int>(keys.size()), axes.data(), layers.data(),
                               pr.data(), with_kernels ? ke.data() : nullptr);
  if (rc == FRW_ESOLVE) throw SolveError(frw_last_error(ctx), 0.0);
  throw_status(ctx, rc);
  for (size_t q = 0; q < keys.size(); ++q) {
    auto g = std::make_shared<DiscreteSGF>();
    g->n = n;
    g->pitch = 1.0;  // canonical unit pitch
    g->probs.assign(pr.begin() + q * P, pr.begin() + (q + 1) * P);
    g->cdf.resize(P);
    double run = 0;
    for (size_t b = 0; b < P; ++b) g->cdf[b] = run += g->probs[b];
    if (with_kernels)
      for (int a = 0; a < 3; ++a)
        g->grad_kernels[a].assign(ke.begin() + (3 * q + a) * P, ke.begin() + (3 * q + a + 1) * P);
    out.push_back(std::move(g));
  }
  return out;
}
}  // namespace

DiscreteSGF solve_canonical(const ProfileKey& key, bool with_kernels, int device) {
  return *solve_keys({key}, with_kernels, device)[0];
}

// ---- cache -------------------------------------------------------------------

std::shared_ptr<const DiscreteSGF> StratifiedSgfCache::store_locked(
    const ProfileKey& key, std::shared_ptr<const DiscreteSGF> sgf) {
  auto it = map_.find(key);
  if (it != map_.end()) {  // first stored result wins
    touch(it->second);
    return it->second.sgf;
  }
  Entry e;
  e.sgf = std::move(sgf);
  touch(e);
  auto out = map_.emplace(key, e).first->second.sgf;
  while (capacity_ > 0 && map_.size() > capacity_) {
    auto victim = map_.begin();
    for (auto jt = map_.begin(); jt != map_.end(); ++jt)
      if (jt->second.used < victim->second.used) victim = jt;
    map_.erase(victim);
  }
  return out;
}

std::shared_ptr<const DiscreteSGF> StratifiedSgfCache::find(const ProfileKey& key) const {
  std::lock_guard<std::mutex> lk(mu_);
  auto it = map_.find(key);
  if (it == map_.end()) return nullptr;
  touch(it->second);
  return it->second.sgf;
}

std::shared_ptr<const DiscreteSGF> StratifiedSgfCache::get(const ProfileKey& key) {
  {
    std::lock_guard<std::mutex> lk(mu_);
    auto it = map_.find(key);
    if (it != map_.end()) {
      ++hits_;
      touch(it->second);
      return it->second.sgf;
    }
    ++misses_;
  }
  if (key.conductor_sig)
    throw std::invalid_argument("canonical_grid: a conductor signature cannot be reconstructed");
  auto sgf = solve_keys({key}, true, device_)[0];
  std::lock_guard<std::mutex> lk(mu_);
  return store_locked(key, std::move(sgf));
}

std::shared_ptr<const DiscreteSGF> StratifiedSgfCache::get(
    const ProfileKey& key, const std::function<DielectricGrid()>& provider) {
  {
    std::lock_guard<std::mutex> lk(mu_);
    auto it = map_.find(key);
    if (it != map_.end()) {
      ++hits_;
      touch(it->second);
      return it->second.sgf;
    }
    ++misses_;
  }
  const DielectricGrid g = provider();
  if (g.tag == GridTag::General)
    throw std::invalid_argument("StratifiedSgfCache::get: the provided grid is General");
  auto sgf = std::make_shared<DiscreteSGF>(solve_sgf(g, true, device_));
  std::lock_guard<std::mutex> lk(mu_);
  return store_locked(key, std::move(sgf));
}

DielectricGrid canonical_grid(const ProfileKey& key) {
  if (key.conductor_sig)
    throw std::invalid_argument("canonical_grid: a conductor signature cannot be reconstructed");
  if (key.n < 1 || static_cast<int>(key.layers.size()) != key.n || key.axis < 0 || key.axis > 2)
    throw std::invalid_argument("canonical_grid: malformed key");
  DielectricGrid g;
  g.n = key.n;
  g.cube = {{0, 0, 0}, key.n / 2.0};  // unit pitch (sgf_cache.cpp:78-96)
  g.eps.resize(static_cast<size_t>(key.n) * key.n * key.n);
  for (int k = 0; k < key.n; ++k)
    for (int j = 0; j < key.n; ++j)
      for (int i = 0; i < key.n; ++i)
        g.eps[g.index(i, j, k)] = key.layers[key.axis == 0 ? i : (key.axis == 1 ? j : k)];
  classify_grid(g);
  return g;
}

void StratifiedSgfCache::solve_many(const std::vector<ProfileKey>& keys, int /*threads*/) {
  // one device batch per lattice size (the reference fans keys out to host threads)
  std::vector<ProfileKey> todo;
  {
    std::lock_guard<std::mutex> lk(mu_);
    for (const auto& k : keys)
      if (!map_.count(k) && std::find(todo.begin(), todo.end(), k) == todo.end()) todo.push_back(k);
    misses_ += todo.size();
  }
  std::stable_sort(todo.begin(), todo.end(),
                   [](const ProfileKey& a, const ProfileKey& b) { return a.n < b.n; });
  for (size_t i = 0; i < todo.size();) {
    size_t j = i;
    while (j < todo.size() && todo[j].n == todo[i].n) ++j;
    const std::vector<ProfileKey> part(todo.begin() + i, todo.begin() + j);
    const auto sol = solve_keys(part, true, device_);
    std::lock_guard<std::mutex> lk(mu_);
    for (size_t q = 0; q < part.size(); ++q) store_locked(part[q], sol[q]);
    i = j;
  }
}

std::shared_ptr<const DiscreteSGF> StratifiedSgfCache::insert(
    const ProfileKey& key, std::shared_ptr<const DiscreteSGF> sgf) {
  std::lock_guard<std::mutex> lk(mu_);
  return store_locked(key, std::move(sgf));
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
  std::vector<std::pair<ProfileKey, std::shared_ptr<const DiscreteSGF>>> out;
  for (const auto& [k, e] : map_) out.emplace_back(k, e.sgf);
  return out;
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
    o.push_back(k.expanded ? 1 : 0);
    o.push_back(k.conductor_sig ? 1 : 0);
    put_u64(o, k.conductor_sig.value_or(0));
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
    key.expanded = r.uint(1) != 0;
    const bool has_sig = r.uint(1) != 0;
    const uint64_t sig = r.uint(8);
    if (has_sig) key.conductor_sig = sig;
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
    // (expanded / conductor-signature keys are kept and saved back; the
    // walk engine's device table takes the plain stratified keys only)
    {
      std::lock_guard<std::mutex> lk(mu_);
      store_locked(key, std::move(sgf));
      ++loaded;
    }
  }
  if (r.pos != buf.size()) throw std::runtime_error("SGF cache: trailing bytes");
  return loaded;
}

}  // namespace frwcap
