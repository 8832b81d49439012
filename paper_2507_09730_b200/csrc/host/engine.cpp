// engine.cpp -- host driver of the device walk engine.
//
// Mirrors the reference's Config / Engine / extract surface
// (proj/include/frwcap/engine.hpp:23-177, proj/src/engine.cpp:37-513):
// the same knobs and validation, the same Gaussian surface and snap
// distance, the same batch/convergence rule and walk-order fold, so a
// caller sees the reference's CapacitanceResult.  The walks themselves run
// on the device through frw_run_walks (include/frw_gpu.h); SGF table misses
// come back through a callback and are solved by StratifiedSgfCache.
#include <algorithm>
#include <cctype>
#include <chrono>
#include <cmath>
#include <limits>
#include <map>
#include <mutex>
#include <thread>
#include <unordered_set>

#include "frwcap.hpp"

namespace frwcap {

namespace {
using Clock = std::chrono::steady_clock;
}

Mode parse_mode(const std::string& name) {
  std::string u(name);
  std::transform(u.begin(), u.end(), u.begin(), [](unsigned char c) { return std::toupper(c); });
  if (u == "FDM") return Mode::FDM;
  if (u == "MW") return Mode::MW;
  if (u == "MWE") return Mode::MWE;
  if (u == "HYBRID-MW") return Mode::HybridMW;
  if (u == "HYBRID-MWE") return Mode::HybridMWE;
  throw std::invalid_argument("unknown mode: " + name);
}

std::string mode_name(Mode m) {
  switch (m) {
    case Mode::FDM: return "FDM";
    case Mode::MW: return "MW";
    case Mode::MWE: return "MWE";
    case Mode::HybridMW: return "HYBRID-MW";
    case Mode::HybridMWE: return "HYBRID-MWE";
  }
  return "?";
}

// engine.cpp:69-82
void Config::validate() const {
  if (grid_n < 2) throw std::invalid_argument("grid_n must be >= 2");
  if (!(expansion >= 1.0)) throw std::invalid_argument("expansion must be >= 1");
  if (!(rel_std_tol > 0.0 && rel_std_tol < 1.0))
    throw std::invalid_argument("rel_std_tol must lie in (0,1)");
  if (min_walks < 1 || max_walks < min_walks)
    throw std::invalid_argument("need 1 <= min_walks <= max_walks");
  if (batch < 1) throw std::invalid_argument("batch must be >= 1");
  if (!(snap_tol > 0.0)) throw std::invalid_argument("snap_tol must be > 0");
  if (hop_cap < 1) throw std::invalid_argument("hop_cap must be >= 1");
  if (!(gaussian_gap_fraction > 0.0 && gaussian_gap_fraction < 1.0))
    throw std::invalid_argument("gaussian_gap_fraction must lie in (0,1)");
  if (grid_n > 128) throw std::invalid_argument("grid_n must be <= 128 on the device");
  if (device_batch < 0) throw std::invalid_argument("device_batch must be >= 0 (0 = auto)");
  for (int d : devices)
    if (d < 0) throw std::invalid_argument("devices: device indices must be >= 0");
}

// engine.cpp:84-124
GaussianSurface gaussian_surface(const Structure& s, double gap_fraction) {
  if (!(gap_fraction > 0.0 && gap_fraction < 1.0))
    throw ValidationError("gaussian gap fraction must lie in (0,1)");
  const Conductor* m = s.find_conductor(s.master_id);
  if (!m) throw ValidationError("master conductor not found");
  double gap = std::numeric_limits<double>::infinity();
  for (int a = 0; a < 3; ++a) {
    gap = std::min(gap, m->box.lo[a] - s.world.lo[a]);
    gap = std::min(gap, s.world.hi[a] - m->box.hi[a]);
  }
  for (const Conductor& c : s.conductors) {
    if (c.id == s.master_id) continue;
    double g = 0;  // Chebyshev gap between disjoint boxes
    for (int a = 0; a < 3; ++a)
      g = std::max(g, std::max(m->box.lo[a] - c.box.hi[a], c.box.lo[a] - m->box.hi[a]));
    gap = std::min(gap, std::max(g, 0.0));
  }
  if (!(gap > 0.0)) throw ValidationError("master touches another conductor or the wall");
  GaussianSurface out;
  const double inflate = gap_fraction * gap;
  for (int a = 0; a < 3; ++a) {
    out.box.lo[a] = m->box.lo[a] - inflate;
    out.box.hi[a] = m->box.hi[a] + inflate;
  }
  const double ex = out.box.hi.x - out.box.lo.x;
  const double ey = out.box.hi.y - out.box.lo.y;
  const double ez = out.box.hi.z - out.box.lo.z;
  const std::array<double, 6> f = {ey * ez, ey * ez, ex * ez, ex * ez, ex * ey, ex * ey};
  double total = 0;
  for (double v : f) total += v;
  double acc = 0;
  for (int i = 0; i < 6; ++i) {
    acc += f[i] / total;
    out.face_cdf[i] = acc;
  }
  out.face_cdf[5] = 1.0;
  out.area_m2 = total * kMetersPerNm * kMetersPerNm;
  return out;
}

const TerminalEstimate* CapacitanceResult::find_terminal(int id) const {
  for (const auto& t : terminals)
    if (t.conductor_id == id) return &t;
  return nullptr;
}

const TerminalEstimate& CapacitanceResult::self() const {
  const TerminalEstimate* t = find_terminal(master_id);
  if (!t) throw std::logic_error("result has no master terminal");
  return *t;
}

// ---- device context ---------------------------------------------------------

void throw_status(frw_ctx* ctx, int rc) {
  if (rc == FRW_OK) return;
  const std::string msg = frw_last_error(ctx);
  switch (rc) {
    case FRW_EINVAL: throw std::invalid_argument(msg);
    case FRW_ESOLVE: throw SolveError(msg, 0.0);
    case FRW_EENGULFED: throw EngulfedStart(msg);
    default: throw std::runtime_error(msg);
  }
}

namespace {
std::mutex g_dev_mu;
std::map<std::pair<int, int>, Device*>& devices() {
  static auto* m = new std::map<std::pair<int, int>, Device*>;  // intentionally leaked:
  return *m;                                                    // no teardown after CUDA exits
}
std::mutex g_tab_mu;  // guards the tables() map (lanes of a multi-device extract)
constexpr int64_t kTallyChunk = 1024;  // walks per device partial tally (frw_walk_chunk_tallies)

struct DeviceTable {
  int n = 0;  // lattice size of the keys currently on the device
  std::unordered_set<ProfileKey, ProfileKeyHash> keys;  // keys already put
  // page-locked staging for per-walk records (two buffers: the host folds
  // one chunk while the device fills the other), kept across extract calls
  frw_walk_record* rec[2] = {nullptr, nullptr};
  size_t rec_cap[2] = {0, 0};
  // per-1024-walk partial tallies (frw_walk_chunk_tallies), same two buffers
  std::vector<double> csum[2], csq[2];
  std::vector<uint64_t> cland[2], cstat[2];
  int64_t nchunks[2] = {0, 0};
};
std::map<frw_ctx*, DeviceTable>& tables() {
  static auto* m = new std::map<frw_ctx*, DeviceTable>;
  return *m;
}
DeviceTable& table_of(frw_ctx* ctx) {
  std::lock_guard<std::mutex> lk(g_tab_mu);
  return tables()[ctx];  // node-based map: the reference stays valid
}

void put_entry(frw_ctx* ctx, const ProfileKey& k, const DiscreteSGF& g) {
  auto& keys = table_of(ctx).keys;
  if (keys.count(k)) return;  // on the device already (frw_sgf_put would skip it too)
  std::vector<double> kern;
  const bool has = !g.grad_kernels[0].empty();
  if (has) {
    kern.reserve(3 * g.probs.size());
    for (const auto& v : g.grad_kernels) kern.insert(kern.end(), v.begin(), v.end());
  }
  throw_status(ctx, frw_sgf_put(ctx, k.n, k.axis, k.layers.data(), g.pitch, g.probs.data(),
                                g.cdf.data(), has ? kern.data() : nullptr));
  keys.insert(k);
}
}  // namespace

Device::Device(int device) {
  const int rc = frw_ctx_create(device, &ctx_);
  if (rc != FRW_OK)
    throw std::runtime_error("cannot open CUDA device " + std::to_string(device) +
                             " (the B200 build has no CPU fallback)");
}

Device::~Device() { frw_ctx_destroy(ctx_); }

void clear_device_tables() {
  std::lock_guard<std::mutex> lk(g_tab_mu);
  for (auto& [ctx, T] : tables()) {
    throw_status(ctx, frw_sgf_clear(ctx));
    T.keys.clear();
    T.n = 0;
  }
}

Device& Device::get(int device, int instance) {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  auto& m = devices();
  const auto key = std::make_pair(device, instance);
  auto it = m.find(key);
  if (it == m.end()) it = m.emplace(key, new Device(device)).first;
  return *it->second;
}

// ---- engine -------------------------------------------------------------------

Engine::Engine(const Structure& s, const Config& cfg, StratifiedSgfCache* cache)
    : s_(s), cfg_(cfg) {
  cfg_.validate();
  s_.validate();
  if (cache) {
    cache_ = cache;
  } else {
    owned_cache_ = std::make_unique<StratifiedSgfCache>();
    cache_ = owned_cache_.get();
  }
  surface_ = gaussian_surface(s_, cfg_.gaussian_gap_fraction);
  const Vec3 he = surface_.box.half_extent();
  snap_ = cfg_.snap_tol * std::max({he.x, he.y, he.z});  // engine.cpp:186-187
  for (size_t i = 0; i < s_.conductors.size(); ++i)
    if (s_.conductors[i].id == s_.master_id) master_slot_ = static_cast<int>(i);
  const std::vector<int> devs = cfg_.devices.empty() ? std::vector<int>{cfg_.device}
                                                     : cfg_.devices;
  std::map<int, int> seen;
  for (int d : devs) ctxs_.push_back(Device::get(d, seen[d]++).ctx());
  ctx_ = ctxs_[0];
}

void Engine::upload(frw_ctx* ctx) const {
  upload_structure(ctx, s_);
  // device table: one lattice size; carry over every cached key of this size
  DeviceTable& T = table_of(ctx);
  if (T.n != cfg_.grid_n) {
    throw_status(ctx, frw_sgf_clear(ctx));
    T.keys.clear();
    T.n = cfg_.grid_n;
  }
  for (const auto& [k, g] : cache_->entries())
    if (k.n == cfg_.grid_n && !k.expanded && !k.conductor_sig) put_entry(ctx, k, *g);
}

frw_walk_params Engine::params() const {
  frw_walk_params p{};
  p.grid_n = cfg_.grid_n;
  switch (cfg_.mode) {
    case Mode::FDM: p.mode = FRW_MODE_FDM; break;
    case Mode::MW: p.mode = FRW_MODE_MW; break;
    case Mode::MWE: p.mode = FRW_MODE_MWE; break;
    case Mode::HybridMWE: p.mode = FRW_MODE_HYBRID_MWE; break;
    default: p.mode = FRW_MODE_HYBRID_MW; break;
  }
  p.expansion = cfg_.expansion;
  p.snap = snap_;
  p.hop_cap = cfg_.hop_cap;
  p.seed = cfg_.seed;
  p.rng_mode = cfg_.rng == RngMode::Philox ? FRW_RNG_PHILOX : FRW_RNG_SPLITMIX_PARITY;
  p.n_slots = 0;
  for (int a = 0; a < 3; ++a) {
    p.gauss_box[a] = surface_.box.lo[a];
    p.gauss_box[3 + a] = surface_.box.hi[a];
  }
  for (int f = 0; f < 6; ++f) p.face_cdf[f] = surface_.face_cdf[f];
  p.area_m2 = surface_.area_m2;
  return p;
}

namespace {
struct MissCtx {
  frw_ctx* ctx;
  StratifiedSgfCache* cache;
  std::string err;
};

// Table misses: keys already in the host cache (e.g. loaded from an SGF1
// file) are uploaded; the rest are solved on the device (frw_sgf_solve),
// stored in the host cache (persistable) and uploaded.
int miss_cb(void* user, int n, int count, const int* axes, const double* layers) {
  auto* m = static_cast<MissCtx*>(user);
  try {
    std::vector<ProfileKey> keys(count), todo;
    for (int q = 0; q < count; ++q) {
      keys[q].n = n;
      keys[q].axis = axes[q];
      keys[q].layers.assign(layers + static_cast<size_t>(q) * n,
                            layers + static_cast<size_t>(q + 1) * n);
      if (!m->cache->find(keys[q])) todo.push_back(keys[q]);
    }
    if (!todo.empty()) {
      const size_t P = 6ull * n * n;
      std::vector<int> ax;
      std::vector<double> lay;
      for (const auto& k : todo) {
        ax.push_back(k.axis);
        lay.insert(lay.end(), k.layers.begin(), k.layers.end());
      }
      std::vector<double> pr(P * todo.size()), ke(3 * P * todo.size());
      throw_status(m->ctx, frw_sgf_solve(m->ctx, n, static_cast<int>(todo.size()), ax.data(),
                                         lay.data(), pr.data(), ke.data()));
      m->cache->count_misses(todo.size());
      for (size_t q = 0; q < todo.size(); ++q) {
        auto g = std::make_shared<DiscreteSGF>();
        g->n = n;
        g->pitch = 1.0;  // canonical unit pitch
        g->probs.assign(pr.begin() + q * P, pr.begin() + (q + 1) * P);
        g->cdf.resize(P);
        double run = 0;
        for (size_t b = 0; b < P; ++b) g->cdf[b] = run += g->probs[b];
        for (int a = 0; a < 3; ++a)
          g->grad_kernels[a].assign(ke.begin() + (3 * q + a) * P, ke.begin() + (3 * q + a + 1) * P);
        m->cache->insert(todo[q], std::move(g));
      }
    }
    for (const auto& k : keys) put_entry(m->ctx, k, *m->cache->find(k));
    return 0;
  } catch (const std::exception& e) {
    m->err = e.what();
    return 1;
  }
}
}  // namespace

std::vector<frw_walk_record> Engine::run_walks(uint64_t begin, int64_t count) {
  upload();
  std::vector<frw_walk_record> rec(count);
  std::vector<double> sum(s_.conductors.size() + 1), sq(sum.size());
  std::vector<uint64_t> landed(sum.size());
  frw_tally t{};
  t.sum = sum.data();
  t.sumsq = sq.data();
  t.landed = landed.data();
  MissCtx mc{ctx_, cache_, {}};
  const frw_walk_params p = params();
  const int rc = frw_run_walks(ctx_, &p, master_slot_, begin, count, miss_cb, &mc, &t, rec.data());
  if (rc != FRW_OK && !mc.err.empty()) throw SolveError(mc.err, 0.0);
  throw_status(ctx_, rc);
  return rec;
}

WalkTally Engine::run_tally(uint64_t begin, int64_t count, bool allreduce) {
  upload();
  const size_t k = s_.conductors.size() + 1;
  WalkTally w;
  w.sum.assign(k, 0.0);
  w.sumsq.assign(k, 0.0);
  w.landed.assign(k, 0);
  frw_tally t{};
  t.sum = w.sum.data();
  t.sumsq = w.sumsq.data();
  t.landed = w.landed.data();
  MissCtx mc{ctx_, cache_, {}};
  const frw_walk_params p = params();
  const int rc = frw_run_walks(ctx_, &p, master_slot_, begin, count, miss_cb, &mc, &t, nullptr);
  if (rc != FRW_OK && !mc.err.empty()) throw SolveError(mc.err, 0.0);
  throw_status(ctx_, rc);
  w.walks = static_cast<uint64_t>(count);
  w.mw_ms = t.mw_ms;
  w.total_ms = t.total_ms;
  if (allreduce) throw_status(ctx_, frw_tally_allreduce(ctx_, nullptr, &t));
  w.mw_jumps = t.mw_jumps;
  w.mw_jump_steps = t.mw_jump_steps;
  w.mw_dense_hops = t.mw_dense_hops;
  w.aborted = t.aborted;
  w.resampled = t.resampled;
  w.mw_steps = t.mw_steps;
  for (int b = 0; b < 4; ++b) {
    w.first[b] = t.first[b];
    w.sub[b] = t.sub[b];
  }
  return w;
}

CapacitanceResult Engine::extract(int /*threads: walks run on the device*/) {
  const auto t_start = Clock::now();
  for (frw_ctx* c : ctxs_) upload(c);
  const size_t nslots = s_.conductors.size() + 1;
  const int master = master_slot_;
  std::vector<double> sum(nslots, 0.0), sumsq(nslots, 0.0);
  std::vector<uint64_t> landed(nslots, 0);
  CapacitanceResult res;
  uint64_t walks = 0;
  bool converged = false;
  double mw_ms = 0, dev_ms = 0;
  const auto misses0 = cache_->stats().misses;

  // engine.cpp:388-420: mean/SE per slot and the stopping rule
  auto estimate = [&](size_t k) {
    const double w = static_cast<double>(walks);
    const double mean = sum[k] / w;
    double se = 0;
    if (walks > 1) se = std::sqrt(std::max(0.0, (sumsq[k] - sum[k] * sum[k] / w) / (w - 1)) / w);
    return std::pair<double, double>(mean, se);
  };
  auto converged_now = [&]() {
    const auto [self, self_se] = estimate(master);
    if (!(self > 0)) return false;
    if (self_se > cfg_.rel_std_tol * self) return false;
    if (cfg_.all_couplings_rule) {
      for (size_t k = 0; k + 1 < nslots; ++k) {
        if (static_cast<int>(k) == master) continue;
        const auto [v, se] = estimate(k);
        if (se > cfg_.rel_std_tol * std::fabs(v)) return false;
      }
      return true;
    }
    size_t big = nslots;
    double big_abs = 0;
    for (size_t k = 0; k < nslots; ++k) {
      if (static_cast<int>(k) == master) continue;
      const double a = std::fabs(sum[k] / static_cast<double>(walks));
      if (a > big_abs) {
        big_abs = a;
        big = k;
      }
    }
    if (big == nslots) return true;
    const auto [v, se] = estimate(big);
    return se <= cfg_.rel_std_tol * std::fabs(v);
  };

  const frw_walk_params p = params();
  // one lane per context: its miss context, tallies, and per-walk records in
  // page-locked memory kept with the context (two buffers: the host folds
  // one wave while the device fills the next)
  struct Lane {
    frw_ctx* ctx;
    DeviceTable* dt;
    MissCtx mc;
    std::vector<double> ts, tq;
    std::vector<uint64_t> tl;
    frw_tally t{};
    int rc = FRW_OK;
    int64_t begin = 0, count = 0;
  };
  std::vector<Lane> lanes;
  for (frw_ctx* c : ctxs_)
    lanes.push_back(Lane{c, &table_of(c), MissCtx{c, cache_, {}},
                         std::vector<double>(nslots), std::vector<double>(nslots),
                         std::vector<uint64_t>(nslots)});
  const long batch = cfg_.batch;
  const long db = cfg_.device_batch > 0 ? cfg_.device_batch
                  : cfg_.min_walks >= cfg_.max_walks ? (1L << 24) : (1L << 22);
  const long dev_batch = std::max<long>(batch, db / batch * batch);
  // fold one chunk's per-walk results in walk order, one reference batch at
  // a time, with the stopping rule after each batch (engine.cpp:378-420)
  auto fold = [&](const frw_walk_record* rec, int64_t chunk) {
    for (int64_t off = 0; off < chunk; off += batch) {
      const int64_t end = std::min<int64_t>(chunk, off + batch);
      for (int64_t i = off; i < end; ++i) {
        const frw_walk_record& r = rec[i];
        sum[r.slot] += r.weight;
        sumsq[r.slot] += r.weight * r.weight;
        ++landed[r.slot];
        res.aborted += r.aborted;
        res.resampled += r.resampled;
        switch (r.branch) {
          case 0: ++res.dispatch.first_stratified; break;
          case 1: ++res.dispatch.first_shrunk; break;
          case 2: ++res.dispatch.first_layered; break;
          case 3: ++res.dispatch.first_homogenized; break;
          default: break;
        }
        res.dispatch.cached += r.cached;
        if (cfg_.mode == Mode::MWE || cfg_.mode == Mode::HybridMWE)
          res.dispatch.microwalk_e += r.microwalk;  // engine.cpp:328 counts every MWE hop
        else if (cfg_.mode == Mode::FDM)
          res.dispatch.fdm += r.microwalk;  // general cubes solved per hop (engine.cpp:312)
        else
          res.dispatch.microwalk += r.microwalk;
        res.mw_steps += r.mw_steps;
      }
      walks += end - off;
      if (walks >= static_cast<uint64_t>(cfg_.min_walks) && converged_now()) {
        converged = true;
        break;
      }
    }
  };
  // The same fold from the device's per-chunk tallies (1024 consecutive walks
  // each, summed in walk order): when reference batches are whole chunks,
  // only ~200 bytes per 1024 walks and slot cross PCIe instead of the
  // records; a batch adds its chunks in order, so the result is the same for
  // every device chunking and device count
  const bool use_chunks = batch % kTallyChunk == 0;
  auto fold_chunks = [&](const DeviceTable& DT, int buf, int64_t chunk) {
    const size_t ns = nslots;
    for (int64_t off = 0; off < chunk; off += batch) {
      const int64_t end = std::min<int64_t>(chunk, off + batch);
      for (int64_t c = off / kTallyChunk; c < (end + kTallyChunk - 1) / kTallyChunk; ++c) {
        for (size_t k = 0; k < ns; ++k) {
          sum[k] += DT.csum[buf][c * ns + k];
          sumsq[k] += DT.csq[buf][c * ns + k];
          landed[k] += DT.cland[buf][c * ns + k];
        }
        const uint64_t* st = &DT.cstat[buf][c * 12];
        res.aborted += st[0];
        res.resampled += st[1];
        res.dispatch.first_stratified += st[2];
        res.dispatch.first_shrunk += st[3];
        res.dispatch.first_layered += st[4];
        res.dispatch.first_homogenized += st[5];
        res.dispatch.cached += st[6];
        if (cfg_.mode == Mode::MWE || cfg_.mode == Mode::HybridMWE)
          res.dispatch.microwalk_e += st[7];
        else if (cfg_.mode == Mode::FDM)
          res.dispatch.fdm += st[7];
        else
          res.dispatch.microwalk += st[7];
        res.mw_steps += st[8];
      }
      walks += end - off;
      if (walks >= static_cast<uint64_t>(cfg_.min_walks) && converged_now()) {
        converged = true;
        break;
      }
    }
  };
  // Device chunks of dev_batch walks (each drains its slot pool through the
  // run-to-completion tail once, so large chunks amortise it), G at a time
  // (one per lane / device, in walk order).  While the devices run wave k+1 a
  // host thread folds wave k in walk order; chunks launched after the
  // stopping rule fired inside an earlier one are discarded, so the result
  // equals the sequential fold for any number of devices.
  //
  // Under a stopping rule with chunk tallies (a fold of ~1 ms per wave) the
  // fold runs before the next wave is sized instead: no speculative wave is
  // thrown away, and once the walk count the rule needs is in sight
  // (SE ~ 1/sqrt(walks): walks * (se / (tol |C|))^2 for the entries the rule
  // tests) the wave is cut to reach it with a 3% margin, in whole reference
  // batches and not below kMinWave.  Only the partition of the one walk
  // sequence into device calls changes: the walks, the fold order and the
  // batch at which the rule fires are the same.
  const bool seq_fold = use_chunks && cfg_.min_walks < cfg_.max_walks;
  constexpr int64_t kMinWave = 1 << 19;
  auto walks_needed = [&]() -> double {
    const double inf = std::numeric_limits<double>::infinity();
    if (walks < 2) return inf;
    auto need = [&](size_t k) {
      const auto [v, se] = estimate(k);
      if (!(std::fabs(v) > 0)) return inf;
      const double r = se / (cfg_.rel_std_tol * std::fabs(v));
      return static_cast<double>(walks) * r * r;
    };
    double n = need(master);
    if (cfg_.all_couplings_rule) {
      for (size_t k = 0; k + 1 < nslots; ++k)
        if (static_cast<int>(k) != master) n = std::max(n, need(k));
      return n;
    }
    size_t big = nslots;
    double big_abs = 0;
    for (size_t k = 0; k < nslots; ++k) {
      if (static_cast<int>(k) == master) continue;
      const double a = std::fabs(sum[k] / static_cast<double>(walks));
      if (a > big_abs) {
        big_abs = a;
        big = k;
      }
    }
    return big == nslots ? n : std::max(n, need(big));
  };
  const int64_t max_walks = cfg_.max_walks;
  int64_t launched = 0;
  int cur = 0;
  std::thread worker;
  auto run_lane = [&](Lane& L, int buf) {
    L.t = frw_tally{};
    L.rc = FRW_OK;
    if (L.count <= 0) return;
    DeviceTable& DT = *L.dt;
    L.t.sum = L.ts.data();
    L.t.sumsq = L.tq.data();
    L.t.landed = L.tl.data();
    if (use_chunks) {
      L.rc = frw_run_walks(L.ctx, &p, master, L.begin, L.count, miss_cb, &L.mc, &L.t, nullptr);
      if (L.rc != FRW_OK) return;
      const size_t nc = (L.count + kTallyChunk - 1) / kTallyChunk;
      DT.csum[buf].resize(nc * nslots);
      DT.csq[buf].resize(nc * nslots);
      DT.cland[buf].resize(nc * nslots);
      DT.cstat[buf].resize(nc * 12);
      int32_t ch = 0;
      L.rc = frw_walk_chunk_tallies(L.ctx, &DT.nchunks[buf], &ch, DT.csum[buf].data(),
                                    DT.csq[buf].data(), DT.cland[buf].data(), DT.cstat[buf].data());
      if (L.rc == FRW_OK && (ch != kTallyChunk || DT.nchunks[buf] != static_cast<int64_t>(nc)))
        L.rc = FRW_ECUDA;
      return;
    }
    if (DT.rec_cap[buf] < static_cast<size_t>(L.count)) {
      if (DT.rec[buf]) frw_host_free(L.ctx, DT.rec[buf]);
      DT.rec[buf] = nullptr;
      DT.rec_cap[buf] = 0;
      void* mem = nullptr;
      L.rc = frw_host_alloc(L.ctx, sizeof(frw_walk_record) * L.count, &mem);
      if (L.rc != FRW_OK) return;
      DT.rec[buf] = static_cast<frw_walk_record*>(mem);
      DT.rec_cap[buf] = L.count;
    }
    L.t.sum = L.ts.data();
    L.t.sumsq = L.tq.data();
    L.t.landed = L.tl.data();
    L.rc = frw_run_walks(L.ctx, &p, master, L.begin, L.count, miss_cb, &L.mc, &L.t, DT.rec[buf]);
  };
  for (;;) {
    int64_t wave = 0;
    int64_t lane_batch = dev_batch;
    if (seq_fold && launched == 0) {
      // a short first wave gives the estimate the later waves are sized from
      const int64_t first = std::max<int64_t>(kMinWave, cfg_.min_walks);
      lane_batch = std::min<int64_t>(dev_batch, (first + batch - 1) / batch * batch);
    } else if (seq_fold && walks >= static_cast<uint64_t>(std::max<long>(cfg_.min_walks, 1))) {
      // (the fold of every earlier wave is complete here)
      const double need = walks_needed() * 1.03 - static_cast<double>(launched);
      const double per_lane = need / static_cast<double>(lanes.size());
      if (per_lane < static_cast<double>(dev_batch)) {
        const int64_t want = std::max<int64_t>(kMinWave, static_cast<int64_t>(std::ceil(std::max(per_lane, 0.0))));
        lane_batch = std::min<int64_t>(dev_batch, (want + batch - 1) / batch * batch);
      }
    }
    for (Lane& L : lanes) {
      L.begin = launched;
      L.count = launched < max_walks ? std::min<int64_t>(lane_batch, max_walks - launched) : 0;
      launched += L.count;
      wave += L.count;
    }
    {
      std::vector<std::thread> th;
      for (size_t g = 1; g < lanes.size(); ++g)
        if (lanes[g].count > 0) th.emplace_back(run_lane, std::ref(lanes[g]), cur);
      run_lane(lanes[0], cur);
      for (auto& x : th) x.join();
    }
    if (worker.joinable()) worker.join();
    // the stopping rule fired inside the wave just folded: this wave was
    // speculative; its results, statistics and errors are discarded
    if (converged || wave == 0) break;
    for (Lane& L : lanes) {
      if (L.rc != FRW_OK && !L.mc.err.empty()) throw SolveError(L.mc.err, 0.0);
      throw_status(L.ctx, L.rc);
      mw_ms += L.t.mw_ms;
      res.mw_jumps += L.t.mw_jumps;
      res.mw_jump_steps += L.t.mw_jump_steps;
      res.mw_dense_hops += L.t.mw_dense_hops;
    }
    {
      // device time of the wave: its slowest lane
      double wave_ms = 0;
      for (const Lane& L : lanes) wave_ms = std::max(wave_ms, L.t.total_ms);
      dev_ms += wave_ms;
    }
    std::vector<std::pair<const frw_walk_record*, int64_t>> parts;
    std::vector<std::pair<const DeviceTable*, int64_t>> cparts;
    for (const Lane& L : lanes)
      if (L.count > 0) {
        parts.emplace_back(L.dt->rec[cur], L.count);
        cparts.emplace_back(L.dt, L.count);
      }
    const int fb = cur;
    if (seq_fold) {
      for (size_t i = 0; i < cparts.size() && !converged; ++i)
        fold_chunks(*cparts[i].first, fb, cparts[i].second);
      if (converged) break;
      cur ^= 1;
      continue;
    }
    worker = std::thread([&fold, &fold_chunks, &converged, use_chunks, parts, cparts, fb] {
      for (size_t i = 0; i < parts.size(); ++i) {
        if (use_chunks)
          fold_chunks(*cparts[i].first, fb, cparts[i].second);
        else
          fold(parts[i].first, parts[i].second);
        if (converged) break;
      }
    });
    cur ^= 1;
  }
  res.master_id = s_.master_id;
  res.walks = walks;
  res.converged = converged;
  const auto st = cache_->stats();
  res.cache_misses = st.misses - misses0;
  const uint64_t lookups = res.dispatch.first_total() + res.dispatch.cached;
  res.cache_hits = lookups > res.cache_misses ? lookups - res.cache_misses : 0;
  for (size_t k = 0; k < nslots; ++k) {
    TerminalEstimate te;
    te.conductor_id = k < s_.conductors.size() ? s_.conductors[k].id : -1;
    const auto [v, se] = estimate(k);
    te.value = v;
    te.std_err = se;
    te.walks_landed = landed[k];
    res.terminals.push_back(te);
  }
  res.t_mw_seconds = mw_ms * 1e-3;
  res.t_device_seconds = dev_ms * 1e-3;
  res.t_total_seconds = std::chrono::duration<double>(Clock::now() - t_start).count();
  return res;
}

CapacitanceResult extract(const Structure& s, const Config& cfg, int threads,
                          StratifiedSgfCache* cache) {
  Engine e(s, cfg, cache);
  return e.extract(threads);
}


// ---- single transitions (engine.cpp:126-148, :201-350) -------------------------
GaussianSample sample_gaussian(const GaussianSurface& g, SplitMix64& rng) {
  const double u = rng.uniform();
  int face = 5;
  for (int f = 0; f < 5; ++f)
    if (u < g.face_cdf[f]) {
      face = f;
      break;
    }
  const int axis = kDirAxis[face];
  const int b1 = axis == 0 ? 1 : 0;
  const int b2 = axis == 2 ? 1 : 2;
  GaussianSample out;
  out.axis = axis;
  out.sign = kDirSign[face];
  out.point[axis] = out.sign < 0 ? g.box.lo[axis] : g.box.hi[axis];
  out.point[b1] = g.box.lo[b1] + rng.uniform() * (g.box.hi[b1] - g.box.lo[b1]);
  out.point[b2] = g.box.lo[b2] + rng.uniform() * (g.box.hi[b2] - g.box.lo[b2]);
  return out;
}

DispatchStats& DispatchStats::operator+=(const DispatchStats& o) {
  first_stratified += o.first_stratified;
  first_shrunk += o.first_shrunk;
  first_layered += o.first_layered;
  first_homogenized += o.first_homogenized;
  cached += o.cached;
  microwalk += o.microwalk;
  microwalk_e += o.microwalk_e;
  fdm += o.fdm;
  return *this;
}

std::vector<std::optional<FirstTransition>> Engine::first_transitions(
    const std::vector<GaussianSample>& g, std::vector<SplitMix64>& rngs,
    DispatchStats& stats) const {
  if (g.size() != rngs.size()) throw std::invalid_argument("first_transitions: one rng per sample");
  upload();
  const int count = static_cast<int>(g.size());
  std::vector<double> pts(3 * g.size());
  std::vector<int32_t> ax(2 * g.size());
  std::vector<uint64_t> st(g.size());
  for (int t = 0; t < count; ++t) {
    for (int a = 0; a < 3; ++a) pts[3 * t + a] = g[t].point[a];
    ax[2 * t] = g[t].axis;
    ax[2 * t + 1] = g[t].sign;
    st[t] = rngs[t].state();
  }
  std::vector<frw_first> out(count);
  MissCtx mc{ctx_, cache_, {}};
  const frw_walk_params p = params();
  const int rc = frw_first_transitions(ctx_, &p, count, pts.data(), ax.data(), st.data(), miss_cb,
                                       &mc, out.data());
  if (rc != FRW_OK && !mc.err.empty()) throw SolveError(mc.err, 0.0);
  throw_status(ctx_, rc);
  std::vector<std::optional<FirstTransition>> res(count);
  for (int t = 0; t < count; ++t) {
    rngs[t].set_state(st[t]);
    if (!out[t].ok) continue;
    FirstTransition f;
    f.point = {out[t].point[0], out[t].point[1], out[t].point[2]};
    f.weight = out[t].weight;
    f.branch = out[t].branch;
    switch (f.branch) {
      case 0: ++stats.first_stratified; break;
      case 1: ++stats.first_shrunk; break;
      case 2: ++stats.first_layered; break;
      default: ++stats.first_homogenized; break;
    }
    res[t] = f;
  }
  return res;
}

std::optional<FirstTransition> Engine::first_transition(const GaussianSample& g, SplitMix64& rng,
                                                        DispatchStats& stats) const {
  std::vector<SplitMix64> r{rng};
  auto res = first_transitions({g}, r, stats);
  rng = r[0];
  return res[0];
}

std::vector<WalkEvent> Engine::transitions(const std::vector<Vec3>& points,
                                           std::vector<SplitMix64>& rngs,
                                           DispatchStats& stats) const {
  if (points.size() != rngs.size()) throw std::invalid_argument("transitions: one rng per point");
  upload();
  const int count = static_cast<int>(points.size());
  std::vector<double> pts(3 * points.size());
  std::vector<uint64_t> st(points.size());
  for (int t = 0; t < count; ++t) {
    for (int a = 0; a < 3; ++a) pts[3 * t + a] = points[t][a];
    st[t] = rngs[t].state();
  }
  std::vector<frw_event> out(count);
  MissCtx mc{ctx_, cache_, {}};
  const frw_walk_params p = params();
  const int rc = frw_transitions(ctx_, &p, count, pts.data(), st.data(), miss_cb, &mc, out.data());
  if (rc != FRW_OK && !mc.err.empty()) throw SolveError(mc.err, 0.0);
  throw_status(ctx_, rc);
  std::vector<WalkEvent> res(count);
  for (int t = 0; t < count; ++t) {
    rngs[t].set_state(st[t]);
    const frw_event& e = out[t];
    WalkEvent& w = res[t];
    if (e.kind == 0) {
      w.kind = WalkEvent::Kind::Continue;
      w.point = {e.point[0], e.point[1], e.point[2]};
    } else if (e.kind == 1) {
      w.kind = WalkEvent::Kind::Terminate;
      w.conductor_id = s_.conductors.at(e.conductor).id;
    } else {
      w.kind = WalkEvent::Kind::TerminateGround;
    }
    switch (e.dispatch) {
      case 0: ++stats.cached; break;
      case 1: ++stats.microwalk; break;
      case 2: ++stats.microwalk_e; break;
      case 3: ++stats.fdm; break;
      default: break;
    }
  }
  return res;
}

WalkEvent Engine::transition(const Vec3& point, SplitMix64& rng, MicroWalkScratch& scratch,
                             DispatchStats& stats, double* t_mw) const {
  (void)scratch;
  const auto t0 = Clock::now();
  std::vector<SplitMix64> r{rng};
  DispatchStats local;
  const WalkEvent e = transitions({point}, r, local)[0];
  if (t_mw && (local.microwalk || local.microwalk_e))
    *t_mw += std::chrono::duration<double>(Clock::now() - t0).count();
  stats += local;
  rng = r[0];
  return e;
}

}  // namespace frwcap
