// ref_capi.cpp -- TEST INFRASTRUCTURE: extern "C" entry points over the
// reference's own, unmodified sources (compiled from /root/reference by
// oracle/Makefile into oracle/_ref/libfrwref.so).  Used only to pin the C
// restatement (oracle/frw_oracle.c) and as the CPU "reference" arm of
// bench.py.  Every function forwards to the reference API it names.
#include <cstdint>
#include <cstring>
#include <exception>
#include <algorithm>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "frwcap/engine.hpp"
#include "frwcap/geometry.hpp"
#include "frwcap/microwalk.hpp"
#include "frwcap/sgf.hpp"
#include "frwcap/sgf_cache.hpp"

using namespace frwcap;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  return -1;
}

Box box6(const double* b) { return {{b[0], b[1], b[2]}, {b[3], b[4], b[5]}}; }

DielectricGrid make_grid(int n, const double* eps, const int32_t* mask,
                         const double* c, double h) {
  DielectricGrid g;
  g.n = n;
  g.cube = {{c[0], c[1], c[2]}, h};
  g.eps.assign(eps, eps + static_cast<size_t>(n) * n * n);
  if (mask) g.conductor_mask.assign(mask, mask + static_cast<size_t>(n) * n * n);
  classify_grid(g);
  return g;
}

void exit_out(const Exit& e, int32_t* panel, int32_t* steps, double* pt,
              int32_t* cond) {
  if (panel) *panel = e.kind == Exit::Kind::Surface ? e.panel : -1;
  if (steps) *steps = e.steps;
  if (pt) {
    pt[0] = e.point.x;
    pt[1] = e.point.y;
    pt[2] = e.point.z;
  }
  if (cond) *cond = e.conductor_id;
}

Config make_config(const double* d, const int64_t* i) {
  // d: expansion, tol, snap_tol, gap_fraction, world_margin
  // i: grid_n, mode, min_walks, max_walks, batch, seed, hop_cap
  Config c;
  c.expansion = d[0];
  c.rel_std_tol = d[1];
  c.snap_tol = d[2];
  c.gaussian_gap_fraction = d[3];
  c.world_margin = d[4];
  c.grid_n = static_cast<int>(i[0]);
  c.mode = static_cast<Mode>(i[1]);
  c.min_walks = i[2];
  c.max_walks = i[3];
  c.batch = static_cast<int>(i[4]);
  c.seed = static_cast<uint64_t>(i[5]);
  c.hop_cap = i[6];
  return c;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// microwalk_transit (microwalk.cpp:188-197) with SplitMix64(seed, stream0+t)
int ref_microwalk_grid_batch(int n, const double* eps, const int32_t* mask,
                             const double* c, double h, uint64_t seed,
                             uint64_t stream0, int64_t count, int step_cap,
                             int threads, int32_t* out_panel,
                             int32_t* out_steps, uint64_t* hist,
                             double* step_sum, double* step_sumsq) {
  try {
    const DielectricGrid g = make_grid(n, eps, mask, c, h);
    if (threads < 1) threads = 1;
    const int bins = 6 * n * n;
    std::vector<std::vector<uint64_t>> hs(threads);
    std::vector<double> ss(threads, 0), sq(threads, 0);
    std::vector<std::exception_ptr> errs(threads);
    auto work = [&](int t, int64_t lo, int64_t hi) {
      try {
        MicroWalkScratch scr;
        if (hist) hs[t].assign(bins, 0);
        for (int64_t k = lo; k < hi; ++k) {
          SplitMix64 rng(seed, stream0 + static_cast<uint64_t>(k));
          const Exit e = microwalk_transit(g, rng, scr, step_cap);
          if (out_panel)
            out_panel[k] = e.kind == Exit::Kind::Surface ? e.panel : -1;
          if (out_steps) out_steps[k] = e.steps;
          if (hist && e.kind == Exit::Kind::Surface) hs[t][e.panel]++;
          ss[t] += e.steps;
          sq[t] += double(e.steps) * e.steps;
        }
      } catch (...) {
        errs[t] = std::current_exception();
      }
    };
    std::vector<std::thread> pool;
    int64_t lo = 0;
    for (int t = 0; t < threads; ++t) {
      const int64_t hi = lo + count / threads + (t < count % threads);
      pool.emplace_back(work, t, lo, hi);
      lo = hi;
    }
    for (auto& th : pool) th.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
    double s1 = 0, s2 = 0;
    for (int t = 0; t < threads; ++t) {
      s1 += ss[t];
      s2 += sq[t];
      if (hist)
        for (int b = 0; b < bins; ++b) hist[b] += hs[t][b];
    }
    if (step_sum) *step_sum = s1;
    if (step_sumsq) *step_sumsq = s2;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---- Structure (geometry.hpp:94-128) ----------------------------------
void* ref_structure_new(int n_cond, const int32_t* ids, const double* cboxes,
                        int n_diel, const double* dboxes, const double* deps,
                        double background, const double* world,
                        int32_t master) {
  auto* s = new Structure;
  for (int i = 0; i < n_cond; ++i) s->conductors.push_back({ids[i], box6(cboxes + 6 * i)});
  for (int i = 0; i < n_diel; ++i) s->dielectrics.push_back({box6(dboxes + 6 * i), deps[i]});
  s->background_eps = background;
  s->world = box6(world);
  s->master_id = master;
  return s;
}

// parse_structure (geometry.cpp:173-251); returns null and sets the error
void* ref_structure_parse(const char* text, double world_margin) {
  try {
    return new Structure(parse_structure(text, world_margin));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_structure_free(void* s) { delete static_cast<Structure*>(s); }

void ref_structure_counts(const void* h, int* n_cond, int* n_diel) {
  const auto* s = static_cast<const Structure*>(h);
  *n_cond = static_cast<int>(s->conductors.size());
  *n_diel = static_cast<int>(s->dielectrics.size());
}

void ref_structure_dump(const void* h, int32_t* ids, double* cboxes,
                        double* dboxes, double* deps, double* background,
                        double* world, int32_t* master) {
  const auto* s = static_cast<const Structure*>(h);
  auto put = [](const Box& b, double* o) {
    for (int a = 0; a < 3; ++a) {
      o[a] = b.lo[a];
      o[3 + a] = b.hi[a];
    }
  };
  for (size_t i = 0; i < s->conductors.size(); ++i) {
    ids[i] = s->conductors[i].id;
    put(s->conductors[i].box, cboxes + 6 * i);
  }
  for (size_t i = 0; i < s->dielectrics.size(); ++i) {
    put(s->dielectrics[i].box, dboxes + 6 * i);
    deps[i] = s->dielectrics[i].eps_r;
  }
  *background = s->background_eps;
  put(s->world, world);
  *master = s->master_id;
}

int ref_permittivity_at(const void* h, const double* p, double* eps) {
  try {
    *eps = static_cast<const Structure*>(h)->permittivity_at({p[0], p[1], p[2]});
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// returns 1 and the id when a conductor is within tol, else 0
int ref_conductor_at(const void* h, const double* p, double tol, int32_t* id) {
  const auto r = static_cast<const Structure*>(h)->conductor_at({p[0], p[1], p[2]}, tol);
  if (!r) return 0;
  *id = *r;
  return 1;
}

int ref_max_free_cube(const void* h, const double* p, double* hw, int32_t* nearest) {
  try {
    const FreeCube f = static_cast<const Structure*>(h)->max_free_cube({p[0], p[1], p[2]});
    *hw = f.half_width;
    *nearest = f.nearest_id ? *f.nearest_id : -1;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// returns axis, -1 when not stratified, -2 on error
int ref_stratified_profile(const void* h, const double* c, double hw, int n,
                           double* layers) {
  try {
    const auto prof = stratified_profile(*static_cast<const Structure*>(h),
                                         {{c[0], c[1], c[2]}, hw}, n);
    if (!prof) return -1;
    for (int t = 0; t < n; ++t) layers[t] = prof->layers[t];
    return prof->axis;
  } catch (const std::exception& e) {
    fail(e);
    return -2;
  }
}

int ref_build_grid(const void* h, const double* c, double hw, int n,
                   int allow_conductors, double* eps, int32_t* mask,
                   int* tag, int* strat_axis) {
  try {
    const DielectricGrid g = build_grid(*static_cast<const Structure*>(h),
                                        {{c[0], c[1], c[2]}, hw}, n,
                                        allow_conductors != 0);
    std::memcpy(eps, g.eps.data(), sizeof(double) * g.eps.size());
    if (mask && g.has_mask())
      std::memcpy(mask, g.conductor_mask.data(), sizeof(int32_t) * g.eps.size());
    *tag = static_cast<int>(g.tag);
    *strat_axis = g.strat_axis;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// microwalk_transit_lazy (microwalk.cpp:199-204), one stream per transit
int ref_microwalk_lazy_batch(const void* h, const double* c, double hw, int n,
                             uint64_t seed, uint64_t stream0, int64_t count,
                             int32_t* panel, int32_t* steps, double* points) {
  try {
    const auto& s = *static_cast<const Structure*>(h);
    const Cube cube{{c[0], c[1], c[2]}, hw};
    MicroWalkScratch scr;
    for (int64_t k = 0; k < count; ++k) {
      SplitMix64 rng(seed, stream0 + static_cast<uint64_t>(k));
      const Exit e = microwalk_transit_lazy(s, cube, n, rng, scr);
      exit_out(e, panel ? panel + k : nullptr, steps ? steps + k : nullptr,
               points ? points + 3 * k : nullptr, nullptr);
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// microwalk_e_transit (microwalk.cpp:206-228); returns -3 on EngulfedStart
int ref_microwalk_e_batch(const void* h, const double* p, double base_hw,
                          double expansion, int n, uint64_t seed,
                          uint64_t stream0, int64_t count, int32_t* panel,
                          int32_t* steps, double* points, int32_t* cond) {
  try {
    const auto& s = *static_cast<const Structure*>(h);
    MicroWalkScratch scr;
    for (int64_t k = 0; k < count; ++k) {
      SplitMix64 rng(seed, stream0 + static_cast<uint64_t>(k));
      const Exit e = microwalk_e_transit(s, {p[0], p[1], p[2]}, base_hw,
                                         expansion, n, rng, scr);
      exit_out(e, panel ? panel + k : nullptr, steps ? steps + k : nullptr,
               points ? points + 3 * k : nullptr, cond ? cond + k : nullptr);
    }
    return 0;
  } catch (const EngulfedStart& e) {
    g_err = e.what();
    return -3;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// solve_sgf (restated in sgf_shim.cpp) on a materialized grid
int ref_solve_sgf(int n, const double* eps, const int32_t* mask,
                  const double* c, double hw, double* probs, double* kernels,
                  double* pitch) {
  try {
    const DiscreteSGF sgf =
        solve_sgf(assemble_system(make_grid(n, eps, mask, c, hw)), kernels != nullptr);
    std::memcpy(probs, sgf.probs.data(), sizeof(double) * sgf.probs.size());
    if (kernels)
      for (int a = 0; a < 3; ++a)
        std::memcpy(kernels + a * sgf.probs.size(), sgf.grad_kernels[a].data(),
                    sizeof(double) * sgf.probs.size());
    if (pitch) *pitch = sgf.pitch;
    return static_cast<int>(sgf.probs.size());
  } catch (const std::exception& e) {
    return fail(e);
  }
}

double ref_expected_steps(int n, const double* eps) {
  const double c[3] = {0, 0, 0};
  try {
    return expected_steps(assemble_system(make_grid(n, eps, nullptr, c, n / 2.0)));
  } catch (const std::exception& e) {
    fail(e);
    return -1;
  }
}

double ref_round_sig(double x, int digits) { return round_sig(x, digits); }

// Engine::extract (engine.cpp:378-507).  Slot arrays hold n_cond+1 entries.
// stats: walks, converged, aborted, resampled, first[4], sub[4], hits, misses
int ref_extract(const void* h, const double* cfg_d, const int64_t* cfg_i,
                int threads, double* value, double* std_err, uint64_t* landed,
                uint64_t* stats, double* times) {
  try {
    const auto& s = *static_cast<const Structure*>(h);
    const CapacitanceResult r = extract(s, make_config(cfg_d, cfg_i), threads);
    for (size_t k = 0; k < r.terminals.size(); ++k) {
      value[k] = r.terminals[k].value;
      std_err[k] = r.terminals[k].std_err;
      landed[k] = r.terminals[k].walks_landed;
    }
    const uint64_t st[14] = {r.walks, r.converged, r.aborted, r.resampled,
                             r.dispatch.first_stratified, r.dispatch.first_shrunk,
                             r.dispatch.first_layered, r.dispatch.first_homogenized,
                             r.dispatch.cached, r.dispatch.microwalk,
                             r.dispatch.microwalk_e, r.dispatch.fdm,
                             r.cache_hits, r.cache_misses};
    std::memcpy(stats, st, sizeof st);
    times[0] = r.t_mw_seconds;
    times[1] = r.t_total_seconds;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// extract() with a process-wide StratifiedSgfCache, so a second call runs
// against a warm table (the CLI's --cache behaviour, cli.cpp:186-193)
static StratifiedSgfCache& warm_cache() {
  static StratifiedSgfCache cache;
  return cache;
}

// loads an SGF1 file into the process-wide cache of ref_extract_warm (the
// CLI's --cache, cli.cpp:186-193, outside any timed region); returns the
// entries loaded or -1
int64_t ref_warm_cache_load(const char* path) {
  try {
    return static_cast<int64_t>(warm_cache().load(path));
  } catch (const std::exception& e) {
    fail(e);
    return -1;
  }
}

int ref_extract_warm(const void* h, const double* cfg_d, const int64_t* cfg_i, int threads,
                     double* value, double* std_err, uint64_t* landed, uint64_t* stats,
                     double* times) {
  StratifiedSgfCache& cache = warm_cache();
  try {
    const auto& s = *static_cast<const Structure*>(h);
    const CapacitanceResult r = extract(s, make_config(cfg_d, cfg_i), threads, &cache);
    for (size_t k = 0; k < r.terminals.size(); ++k) {
      value[k] = r.terminals[k].value;
      std_err[k] = r.terminals[k].std_err;
      landed[k] = r.terminals[k].walks_landed;
    }
    const uint64_t st[14] = {r.walks, r.converged, r.aborted, r.resampled,
                             r.dispatch.first_stratified, r.dispatch.first_shrunk,
                             r.dispatch.first_layered, r.dispatch.first_homogenized,
                             r.dispatch.cached, r.dispatch.microwalk,
                             r.dispatch.microwalk_e, r.dispatch.fdm,
                             r.cache_hits, r.cache_misses};
    std::memcpy(stats, st, sizeof st);
    times[0] = r.t_mw_seconds;
    times[1] = r.t_total_seconds;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Engine::extract with a caller-visible cache: cache_in (SGF1, may be null)
// is loaded first -- the CLI's --cache behaviour (cli.cpp:186-193) -- and
// the cache is saved to cache_out (may be null) afterwards
int ref_extract_cache(const void* h, const double* cfg_d, const int64_t* cfg_i, int threads,
                      const char* cache_in, const char* cache_out, double* value,
                      double* std_err, uint64_t* landed, uint64_t* stats, double* times) {
  try {
    const auto& s = *static_cast<const Structure*>(h);
    StratifiedSgfCache cache;
    if (cache_in && *cache_in) cache.load(cache_in);
    const Config cfg = make_config(cfg_d, cfg_i);
    const CapacitanceResult r = extract(s, cfg, threads, &cache);
    for (size_t k = 0; k < r.terminals.size(); ++k) {
      value[k] = r.terminals[k].value;
      std_err[k] = r.terminals[k].std_err;
      landed[k] = r.terminals[k].walks_landed;
    }
    const uint64_t st[14] = {r.walks, r.converged, r.aborted, r.resampled,
                             r.dispatch.first_stratified, r.dispatch.first_shrunk,
                             r.dispatch.first_layered, r.dispatch.first_homogenized,
                             r.dispatch.cached, r.dispatch.microwalk,
                             r.dispatch.microwalk_e, r.dispatch.fdm,
                             r.cache_hits, r.cache_misses};
    std::memcpy(stats, st, sizeof st);
    times[0] = r.t_mw_seconds;
    times[1] = r.t_total_seconds;
    if (cache_out && *cache_out) cache.save(cache_out, cfg.grid_n);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Per-walk records, restating the 20-line Engine::run_walk
// (engine.cpp:352-376, private) over the public first_transition/transition.
// Walks [w0, w0+count) on `threads` threads (contiguous ranges, as
// engine.cpp:437-458 splits a batch); the engine's StratifiedSgfCache starts
// from cache_in (SGF1, may be null) and is saved to cache_out (may be null)
// afterwards -- the reference's own solved tables, for injection into the
// device table.
static int run_walks_impl(const void* h, const double* cfg_d, const int64_t* cfg_i,
                          uint64_t w0, int64_t count, int threads, const char* cache_in,
                          const char* cache_out, int32_t* slot, double* weight,
                          uint8_t* aborted) {
  try {
    const auto& s = *static_cast<const Structure*>(h);
    const Config cfg = make_config(cfg_d, cfg_i);
    StratifiedSgfCache cache;
    if (cache_in && *cache_in) cache.load(cache_in);
    Engine eng(s, cfg, &cache);
    const int ground = static_cast<int>(s.conductors.size());
    auto slot_of = [&](int id) {
      for (size_t i = 0; i < s.conductors.size(); ++i)
        if (s.conductors[i].id == id) return static_cast<int>(i);
      return ground;
    };
    // one walk: Engine::run_walk (engine.cpp:352-376)
    auto walk = [&](int64_t k, MicroWalkScratch& scr, DispatchStats& ds) {
      SplitMix64 rng(cfg.seed, w0 + static_cast<uint64_t>(k));
      std::optional<FirstTransition> first;
      for (int a = 0; a < 100 && !first; ++a)
        first = eng.first_transition(sample_gaussian(eng.surface(), rng), rng, ds);
      slot[k] = ground;
      weight[k] = 0;
      aborted[k] = 1;
      if (!first) return;
      weight[k] = first->weight;
      Vec3 p = first->point;
      for (long hop = 0; hop < cfg.hop_cap; ++hop) {
        const WalkEvent ev = eng.transition(p, rng, scr, ds);
        if (ev.kind == WalkEvent::Kind::Terminate) {
          slot[k] = slot_of(ev.conductor_id);
          aborted[k] = 0;
          return;
        }
        if (ev.kind == WalkEvent::Kind::TerminateGround) {
          aborted[k] = 0;
          return;
        }
        p = ev.point;
      }
    };
    const int nt = std::max(1, threads);
    std::vector<std::thread> pool;
    std::vector<std::string> errs(nt);
    for (int t = 0; t < nt; ++t)
      pool.emplace_back([&, t] {
        try {
          MicroWalkScratch scr;
          DispatchStats ds;
          for (int64_t k = count * t / nt, hi = count * (t + 1) / nt; k < hi; ++k)
            walk(k, scr, ds);
        } catch (const std::exception& e) {
          errs[t] = e.what();
        }
      });
    for (auto& th : pool) th.join();
    for (const auto& e : errs)
      if (!e.empty()) throw std::runtime_error(e);
    if (cache_out && *cache_out) cache.save(cache_out, cfg.grid_n);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_run_walks(const void* h, const double* cfg_d, const int64_t* cfg_i,
                  uint64_t w0, int64_t count, int32_t* slot, double* weight,
                  uint8_t* aborted) {
  return run_walks_impl(h, cfg_d, cfg_i, w0, count, 1, nullptr, nullptr, slot, weight, aborted);
}

int ref_run_walks_cache(const void* h, const double* cfg_d, const int64_t* cfg_i,
                        uint64_t w0, int64_t count, int threads, const char* cache_in,
                        const char* cache_out, int32_t* slot, double* weight,
                        uint8_t* aborted) {
  return run_walks_impl(h, cfg_d, cfg_i, w0, count, threads, cache_in, cache_out, slot, weight,
                        aborted);
}

// StratifiedSgfCache::get for each key, then save (sgf_cache.cpp:98-131,
// :210-250): an SGF1 file written by the reference's own cache code
int ref_cache_save(int n, int count, const int32_t* axes, const double* layers,
                   const char* path) {
  try {
    StratifiedSgfCache cache;
    for (int q = 0; q < count; ++q) {
      const std::vector<double> lay(layers + static_cast<size_t>(q) * n,
                                    layers + static_cast<size_t>(q + 1) * n);
      cache.get(profile_key(n, axes[q], lay));
    }
    cache.save(path, n);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// loads an SGF1 file with the reference's cache and returns the probs of
// one key (n*n*6 doubles) -- reads files written by the B200 build
int ref_cache_load_probs(const char* path, int n, int axis, const double* layers,
                         double* probs, int64_t* loaded) {
  try {
    StratifiedSgfCache cache;
    *loaded = static_cast<int64_t>(cache.load(path));
    const auto g = cache.find(profile_key(n, axis, std::vector<double>(layers, layers + n)));
    if (!g) return -2;
    std::copy(g->probs.begin(), g->probs.end(), probs);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"
