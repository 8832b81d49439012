// py_module.cpp -- pybind11 module `_core` of the B200 build.
//
// Same names, keyword options, result dictionaries and error mapping as the
// reference module (proj/bindings/py_module.cpp:20-224); the work runs on
// the device.  B200-only extras are prefixed or documented as such.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <cmath>
#include <sstream>

#include "frwcap.hpp"

namespace py = pybind11;
using namespace frwcap;

namespace {

// py_module.cpp:20-57 (+ B200 knobs rng, all_couplings, device_batch, device, devices)
Config config_from_kwargs(const py::kwargs& kw, int& threads) {
  Config cfg;
  threads = 0;
  for (const auto& item : kw) {
    const std::string key = py::cast<std::string>(item.first);
    const py::handle v = item.second;
    if (key == "grid_n") cfg.grid_n = py::cast<int>(v);
    else if (key == "expansion") cfg.expansion = py::cast<double>(v);
    else if (key == "mode") cfg.mode = parse_mode(py::cast<std::string>(v));
    else if (key == "tol") cfg.rel_std_tol = py::cast<double>(v);
    else if (key == "min_walks") cfg.min_walks = py::cast<long>(v);
    else if (key == "max_walks") cfg.max_walks = py::cast<long>(v);
    else if (key == "batch") cfg.batch = py::cast<long>(v);
    else if (key == "seed") cfg.seed = py::cast<uint64_t>(v);
    else if (key == "snap_tol") cfg.snap_tol = py::cast<double>(v);
    else if (key == "hop_cap") cfg.hop_cap = py::cast<long>(v);
    else if (key == "gaussian_gap_fraction") cfg.gaussian_gap_fraction = py::cast<double>(v);
    else if (key == "world_margin") cfg.world_margin = py::cast<double>(v);
    else if (key == "threads") threads = py::cast<int>(v);
    else if (key == "rng") {
      const std::string r = py::cast<std::string>(v);
      if (r == "philox") cfg.rng = RngMode::Philox;
      else if (r == "splitmix") cfg.rng = RngMode::SplitMixParity;
      else throw py::value_error("rng must be 'philox' or 'splitmix'");
    } else if (key == "all_couplings") cfg.all_couplings_rule = py::cast<bool>(v);
    else if (key == "device_batch") cfg.device_batch = py::cast<long>(v);
    else if (key == "device") cfg.device = py::cast<int>(v);
    else if (key == "devices") cfg.devices = py::cast<std::vector<int>>(v);
    else throw py::value_error("unknown option: " + key);
  }
  cfg.validate();
  return cfg;
}


// per-transit Exit fields as numpy arrays; kind -1 marks EngulfedStart
py::dict exits_dict(const std::vector<Exit>& ex, const std::vector<SplitMix64>& rngs) {
  const size_t cnt = ex.size();
  py::array_t<int32_t> kind(cnt), panel(cnt), cond(cnt), dir(cnt), steps(cnt);
  py::array_t<int32_t> voxel({cnt, static_cast<size_t>(3)});
  py::array_t<double> point({cnt, static_cast<size_t>(3)});
  py::array_t<uint64_t> state(cnt);
  for (size_t t = 0; t < cnt; ++t) {
    const Exit& e = ex[t];
    const bool engulfed = e.kind == Exit::Kind::Conductor && e.conductor_id < 0;
    kind.mutable_at(t) = engulfed ? -1 : (e.kind == Exit::Kind::Surface ? 0 : 1);
    panel.mutable_at(t) = e.panel;
    cond.mutable_at(t) = e.conductor_id;
    dir.mutable_at(t) = e.dir;
    steps.mutable_at(t) = e.steps;
    for (int a = 0; a < 3; ++a) {
      voxel.mutable_at(t, a) = e.voxel[a];
      point.mutable_at(t, a) = e.point[a];
    }
    state.mutable_at(t) = rngs[t].state();
  }
  py::dict d;
  d["kind"] = kind;
  d["panel"] = panel;
  d["cond"] = cond;
  d["dir"] = dir;
  d["steps"] = steps;
  d["voxel"] = voxel;
  d["point"] = point;
  d["state"] = state;
  return d;
}

// py_module.cpp:59-98
py::dict result_to_dict(const CapacitanceResult& r) {
  py::list terms;
  for (const auto& t : r.terminals) {
    py::dict e;
    e["conductor_id"] = t.conductor_id;
    e["capacitance_farads"] = t.value;
    e["std_err_farads"] = t.std_err;
    e["walks_landed"] = t.walks_landed;
    terms.append(e);
  }
  py::dict first, sub, dispatch, cache, d;
  first["stratified"] = r.dispatch.first_stratified;
  first["shrunk"] = r.dispatch.first_shrunk;
  first["layered"] = r.dispatch.first_layered;
  first["homogenized"] = r.dispatch.first_homogenized;
  sub["cached"] = r.dispatch.cached;
  sub["microwalk"] = r.dispatch.microwalk;
  sub["microwalk_e"] = r.dispatch.microwalk_e;
  sub["fdm"] = r.dispatch.fdm;
  dispatch["first"] = first;
  dispatch["subsequent"] = sub;
  cache["hits"] = r.cache_hits;
  cache["misses"] = r.cache_misses;
  d["master_id"] = r.master_id;
  d["terminals"] = terms;
  d["walks"] = r.walks;
  d["converged"] = r.converged;
  d["aborted"] = r.aborted;
  d["resampled"] = r.resampled;
  d["dispatch_stats"] = dispatch;
  d["cache"] = cache;
  d["t_mw_seconds"] = r.t_mw_seconds;
  d["t_total_seconds"] = r.t_total_seconds;
  d["mw_steps"] = r.mw_steps;                   // B200 extra
  d["mw_jumps"] = r.mw_jumps;                   // B200 extra
  d["mw_jump_steps"] = r.mw_jump_steps;         // B200 extra: steps the jumps stand for
  d["mw_dense_hops"] = r.mw_dense_hops;         // B200 extra: hops with > 64 boxes in the cube
  d["t_device_seconds"] = r.t_device_seconds;   // B200 extra
  return d;
}

StratifiedSgfCache& shared_cache() {
  static auto* c = new StratifiedSgfCache;  // process-wide, like a CLI --cache
  return *c;
}

py::dict extract_structure(const Structure& s, const Config& cfg, int threads) {
  CapacitanceResult res;
  {
    py::gil_scoped_release release;
    res = extract(s, cfg, threads, &shared_cache());
  }
  return result_to_dict(res);
}

}  // namespace

PYBIND11_MODULE(_core, m) {
  m.doc() = "floating random walk capacitance extraction (B200 device build)";

  m.def(
      "extract_json",
      [](const std::string& text, const py::kwargs& kw) {
        int threads = 0;
        const Config cfg = config_from_kwargs(kw, threads);
        return extract_structure(parse_structure(text, cfg.world_margin), cfg, threads);
      },
      py::arg("structure_json"),
      "Extract the master conductor's capacitance row from a structure given as JSON text.");

  m.def(
      "extract_file",
      [](const std::string& path, const py::kwargs& kw) {
        int threads = 0;
        const Config cfg = config_from_kwargs(kw, threads);
        return extract_structure(parse_structure_file(path, cfg.world_margin), cfg, threads);
      },
      py::arg("path"), "Extract the master conductor's capacitance row from a structure file.");

  m.def(
      "reference_capacitance_file",
      [](const std::string& path, int resolution, double world_margin) {
        const Structure s = parse_structure_file(path, world_margin);
        ReferenceSolution ref;
        {
          py::gil_scoped_release release;
          ref = reference_capacitance(s, resolution);
        }
        // py_module.cpp:110-125
        py::list ids;
        for (int id : ref.terminal_ids) ids.append(id);
        py::list rows;
        const int T = static_cast<int>(ref.terminal_ids.size());
        for (int i = 0; i < T; ++i) {
          py::list row;
          for (int j = 0; j < T; ++j) row.append(ref.at(i, j));
          rows.append(row);
        }
        py::dict d;
        d["terminal_ids"] = ids;
        d["capacitance_farads"] = rows;
        d["residual"] = ref.residual;
        return d;
      },
      py::arg("path"), py::arg("resolution") = 48, py::arg("world_margin") = 5.0);

  // oracle.cpp:296-310: C = eps0 * area / sum(d_k / eps_k)
  m.def(
      "analytic_plate_capacitance",
      [](const std::vector<std::pair<double, double>>& layers, double area_m2) {
        if (layers.empty()) throw std::invalid_argument("analytic_plate_capacitance: no layers");
        double sum = 0;
        for (const auto& [d, e] : layers) {
          if (!(d > 0) || !(e > 0))
            throw std::invalid_argument("analytic_plate_capacitance: nonpositive layer");
          sum += d * kMetersPerNm / e;
        }
        return kEps0 * area_m2 / sum;
      },
      py::arg("layers"), py::arg("area_m2"));

  // py_module.cpp:172-189: TV distance of device transits vs the solved law
  m.def(
      "transit_tv",
      [](int n, uint64_t grid_seed, long samples, uint64_t sample_seed) {
        py::gil_scoped_release release;
        // py_module.cpp:176-193: random voxel grid, exact solve, transits
        SplitMix64 g(grid_seed, 0);
        const DielectricGrid grid = random_voxel_grid(n, g);
        const DiscreteSGF sgf = solve_sgf(grid, false);
        const TransitBatch b = microwalk_transit_batch(n, grid.eps, {0, 0, 0}, n / 2.0, sample_seed,
                                                       0, samples, RngMode::Philox, false);
        double tv = 0;
        for (size_t q = 0; q < sgf.probs.size(); ++q)
          tv += std::fabs(static_cast<double>(b.hist[q]) / samples - sgf.probs[q]);
        return tv / 2;
      },
      py::arg("n"), py::arg("grid_seed"), py::arg("samples"), py::arg("sample_seed"));

  m.def(
      "expected_steps_uniform",
      [](int n) {
        py::gil_scoped_release release;
        DielectricGrid g;
        g.n = n;
        g.cube = {{0, 0, 0}, n / 2.0};
        g.eps.assign(static_cast<size_t>(n) * n * n, 1.0);
        return expected_steps(g);
      },
      py::arg("n"));

  // the reference CLI in-process (cli.hpp run_cli): (rc, stdout, stderr)
  m.def(
      "run_cli",
      [](const std::vector<std::string>& args) -> py::tuple {
        std::ostringstream out, err;
        int rc;
        {
          py::gil_scoped_release release;
          rc = run_cli(args, out, err);
        }
        return py::make_tuple(rc, out.str(), err.str());
      },
      py::arg("args"));

  // ---- B200 extras ---------------------------------------------------------
  m.def(
      "run_walks_json",
      [](const std::string& text, uint64_t begin, int64_t count, const py::kwargs& kw) {
        int threads = 0;
        const Config cfg = config_from_kwargs(kw, threads);
        const Structure s = parse_structure(text, cfg.world_margin);
        std::vector<frw_walk_record> rec;
        {
          py::gil_scoped_release release;
          Engine e(s, cfg, &shared_cache());
          rec = e.run_walks(begin, count);
        }
        py::array_t<int32_t> slot(count);
        py::array_t<double> w(count);
        py::array_t<uint8_t> ab(count);
        py::array_t<uint32_t> mw(count);
        py::array_t<uint64_t> steps(count);
        for (int64_t i = 0; i < count; ++i) {
          slot.mutable_at(i) = rec[i].slot;
          w.mutable_at(i) = rec[i].weight;
          ab.mutable_at(i) = rec[i].aborted;
          mw.mutable_at(i) = rec[i].microwalk;
          steps.mutable_at(i) = rec[i].mw_steps;
        }
        py::dict d;
        d["slot"] = slot;
        d["weight"] = w;
        d["aborted"] = ab;
        d["microwalk"] = mw;
        d["mw_steps"] = steps;
        return d;
      },
      py::arg("structure_json"), py::arg("begin"), py::arg("count"),
      "Per-walk outcomes of walks [begin, begin+count) (parity tests).");


  // ---- multi-GPU (paper_2507_09730_b200/dist.py) ----------
  m.def(
      "run_walks_tally",
      [](const std::string& text, uint64_t begin, int64_t count, bool allreduce,
         const py::kwargs& kw) {
        int threads = 0;
        const Config cfg = config_from_kwargs(kw, threads);
        const Structure s = parse_structure(text, cfg.world_margin);
        WalkTally t;
        {
          py::gil_scoped_release release;
          Engine e(s, cfg, &shared_cache());
          t = e.run_tally(begin, count, allreduce);
        }
        py::dict d;
        d["sum"] = py::array_t<double>(t.sum.size(), t.sum.data());
        d["sumsq"] = py::array_t<double>(t.sumsq.size(), t.sumsq.data());
        d["landed"] = py::array_t<uint64_t>(t.landed.size(), t.landed.data());
        d["walks"] = t.walks;
        d["aborted"] = t.aborted;
        d["resampled"] = t.resampled;
        d["first"] = std::vector<uint64_t>(t.first, t.first + 4);
        d["sub"] = std::vector<uint64_t>(t.sub, t.sub + 4);
        d["mw_steps"] = t.mw_steps;
        d["mw_jumps"] = t.mw_jumps;
        d["mw_jump_steps"] = t.mw_jump_steps;
        d["mw_dense_hops"] = t.mw_dense_hops;
        d["t_mw_seconds"] = t.mw_ms * 1e-3;
        d["t_device_seconds"] = t.total_ms * 1e-3;
        py::list ids;
        for (const auto& c : s.conductors) ids.append(c.id);
        d["conductor_ids"] = ids;
        d["master_id"] = s.master_id;
        return d;
      },
      py::arg("structure_json"), py::arg("begin"), py::arg("count"), py::arg("allreduce") = false,
      "Device tallies of walks [begin, begin+count); allreduce=True sums them over the ranks "
      "of the NCCL communicator set up by nccl_init (frw_tally_allreduce).");
  m.def("nccl_unique_id", []() {
    char id[128];
    if (frw_nccl_unique_id(id) != FRW_OK) throw std::runtime_error("ncclGetUniqueId failed");
    return py::bytes(id, sizeof id);
  });
  m.def(
      "nccl_init",
      [](int device, const py::bytes& uid, int nranks, int rank) {
        const std::string u = uid;
        if (u.size() != 128) throw py::value_error("nccl_init: the unique id has 128 bytes");
        frw_ctx* ctx = Device::get(device).ctx();
        py::gil_scoped_release release;
        throw_status(ctx, frw_nccl_init(ctx, u.data(), nranks, rank));
      },
      py::arg("device"), py::arg("unique_id"), py::arg("nranks"), py::arg("rank"));

  m.def(
      "walks_by_transitions",
      [](const std::string& text, uint64_t begin, int64_t count, bool single,
         const py::kwargs& kw) {
        // run_walk (engine.cpp:352-376) composed from Engine::first_transition
        // and Engine::transition, all walks in lockstep (or one call each)
        int threads = 0;
        const Config cfg = config_from_kwargs(kw, threads);
        const Structure s = parse_structure(text, cfg.world_margin);
        const int ground = static_cast<int>(s.conductors.size());
        auto slot_of = [&](int id) {
          for (size_t i = 0; i < s.conductors.size(); ++i)
            if (s.conductors[i].id == id) return static_cast<int>(i);
          return ground;
        };
        std::vector<int32_t> slot(count, ground);
        std::vector<double> weight(count, 0.0);
        std::vector<uint8_t> aborted(count, 0);
        DispatchStats stats;
        {
          py::gil_scoped_release release;
          Engine e(s, cfg, &shared_cache());
          std::vector<SplitMix64> rng(count);
          for (int64_t w = 0; w < count; ++w) rng[w] = SplitMix64(cfg.seed, begin + w);
          std::vector<int64_t> live(count);
          for (int64_t w = 0; w < count; ++w) live[w] = w;
          std::vector<Vec3> pos(count);
          for (int attempt = 0; attempt < 100 && !live.empty(); ++attempt) {
            std::vector<GaussianSample> g;
            std::vector<SplitMix64> r;
            for (int64_t w : live) {
              g.push_back(sample_gaussian(e.surface(), rng[w]));
              r.push_back(rng[w]);
            }
            std::vector<std::optional<FirstTransition>> f;
            if (single) {
              for (size_t q = 0; q < g.size(); ++q) f.push_back(e.first_transition(g[q], r[q], stats));
            } else {
              f = e.first_transitions(g, r, stats);
            }
            std::vector<int64_t> next;
            for (size_t q = 0; q < live.size(); ++q) {
              const int64_t w = live[q];
              rng[w] = r[q];
              if (f[q]) {
                weight[w] = f[q]->weight;
                pos[w] = f[q]->point;
              } else {
                next.push_back(w);
              }
            }
            live.swap(next);
          }
          for (int64_t w : live) aborted[w] = 1;  // resample cap: ground, weight 0
          std::vector<int64_t> act;
          for (int64_t w = 0; w < count; ++w)
            if (!aborted[w]) act.push_back(w);
          MicroWalkScratch scr;
          for (long hop = 0; hop < cfg.hop_cap && !act.empty(); ++hop) {
            std::vector<Vec3> p;
            std::vector<SplitMix64> r;
            for (int64_t w : act) {
              p.push_back(pos[w]);
              r.push_back(rng[w]);
            }
            std::vector<WalkEvent> ev;
            if (single) {
              for (size_t q = 0; q < p.size(); ++q) ev.push_back(e.transition(p[q], r[q], scr, stats));
            } else {
              ev = e.transitions(p, r, stats);
            }
            std::vector<int64_t> next;
            for (size_t q = 0; q < act.size(); ++q) {
              const int64_t w = act[q];
              rng[w] = r[q];
              if (ev[q].kind == WalkEvent::Kind::Terminate) {
                slot[w] = slot_of(ev[q].conductor_id);
              } else if (ev[q].kind == WalkEvent::Kind::TerminateGround) {
                slot[w] = ground;
              } else {
                pos[w] = ev[q].point;
                next.push_back(w);
              }
            }
            act.swap(next);
          }
          for (int64_t w : act) aborted[w] = 1;  // hop cap
        }
        py::dict d;
        d["slot"] = py::array_t<int32_t>(count, slot.data());
        d["weight"] = py::array_t<double>(count, weight.data());
        d["aborted"] = py::array_t<uint8_t>(count, aborted.data());
        py::dict st;
        st["first_stratified"] = stats.first_stratified;
        st["first_shrunk"] = stats.first_shrunk;
        st["first_layered"] = stats.first_layered;
        st["first_homogenized"] = stats.first_homogenized;
        st["cached"] = stats.cached;
        st["microwalk"] = stats.microwalk;
        st["microwalk_e"] = stats.microwalk_e;
        d["stats"] = st;
        return d;
      },
      py::arg("structure_json"), py::arg("begin"), py::arg("count"), py::arg("single") = false);

  m.def(
      "transitions_json",
      [](const std::string& text, py::array_t<double, py::array::c_style | py::array::forcecast> pts,
         py::array_t<uint64_t, py::array::c_style | py::array::forcecast> states,
         const py::kwargs& kw) {
        // Engine::transitions (batched Engine::transition, engine.hpp:156-159)
        int threads = 0;
        const Config cfg = config_from_kwargs(kw, threads);
        const Structure s = parse_structure(text, cfg.world_margin);
        const size_t cnt = states.size();
        if (pts.size() != 3 * cnt) throw py::value_error("points must be [count][3]");
        std::vector<Vec3> p(cnt);
        std::vector<SplitMix64> r(cnt);
        for (size_t t = 0; t < cnt; ++t) {
          p[t] = {pts.data()[3 * t], pts.data()[3 * t + 1], pts.data()[3 * t + 2]};
          r[t].set_state(states.data()[t]);
        }
        std::vector<WalkEvent> ev;
        DispatchStats st;
        {
          py::gil_scoped_release release;
          Engine e(s, cfg, &shared_cache());
          ev = e.transitions(p, r, st);
        }
        py::array_t<int32_t> kind(cnt), cond(cnt);
        py::array_t<double> point({cnt, static_cast<size_t>(3)});
        py::array_t<uint64_t> state(cnt);
        for (size_t t = 0; t < cnt; ++t) {
          kind.mutable_at(t) = static_cast<int>(ev[t].kind);
          cond.mutable_at(t) = ev[t].conductor_id;
          for (int a = 0; a < 3; ++a) point.mutable_at(t, a) = ev[t].point[a];
          state.mutable_at(t) = r[t].state();
        }
        py::dict d;
        d["kind"] = kind;
        d["conductor_id"] = cond;
        d["point"] = point;
        d["state"] = state;
        py::dict sd;
        sd["cached"] = st.cached;
        sd["microwalk"] = st.microwalk;
        sd["microwalk_e"] = st.microwalk_e;
        sd["fdm"] = st.fdm;
        d["stats"] = sd;
        return d;
      },
      py::arg("structure_json"), py::arg("points"), py::arg("states"));

  // single-transit API (microwalk.hpp:70-100) -- test and integration hooks
  m.def(
      "transits_grid",
      [](py::array_t<double, py::array::c_style | py::array::forcecast> eps,
         std::vector<double> center, double half_width,
         py::array_t<uint64_t, py::array::c_style | py::array::forcecast> states, py::object mask,
         bool single, int step_cap) {
        DielectricGrid g;
        g.n = static_cast<int>(std::lround(std::cbrt(static_cast<double>(eps.size()))));
        g.cube = {{center.at(0), center.at(1), center.at(2)}, half_width};
        g.eps.assign(eps.data(), eps.data() + eps.size());
        if (!mask.is_none()) {
          auto mk = py::cast<py::array_t<int32_t, py::array::c_style | py::array::forcecast>>(mask);
          g.conductor_mask.assign(mk.data(), mk.data() + mk.size());
        }
        std::vector<SplitMix64> rngs(states.size());
        for (size_t t = 0; t < rngs.size(); ++t) rngs[t].set_state(states.data()[t]);
        std::vector<Exit> ex;
        {
          py::gil_scoped_release release;
          if (single) {
            MicroWalkScratch scr;
            for (auto& r : rngs) ex.push_back(microwalk_transit(g, r, scr, step_cap));
          } else {
            ex = microwalk_transits(g, rngs, step_cap);
          }
        }
        return exits_dict(ex, rngs);
      },
      py::arg("eps"), py::arg("center"), py::arg("half_width"), py::arg("states"),
      py::arg("mask") = py::none(), py::arg("single") = false, py::arg("step_cap") = 0);

  m.def(
      "transits_structure",
      [](const std::string& text, py::array_t<double, py::array::c_style | py::array::forcecast> cubes,
         int n, bool expanded, double expansion,
         py::array_t<uint64_t, py::array::c_style | py::array::forcecast> states, bool single,
         int step_cap) {
        const Structure s = parse_structure(text);
        const size_t cnt = states.size();
        if (cubes.size() != 4 * cnt) throw py::value_error("cubes must be [count][4]");
        std::vector<SplitMix64> rngs(cnt);
        for (size_t t = 0; t < cnt; ++t) rngs[t].set_state(states.data()[t]);
        std::vector<Exit> ex(cnt);
        const double* c = cubes.data();
        {
          py::gil_scoped_release release;
          if (single) {
            // expanded: cubes hold (point, base half width) as for microwalk_e_transit
            MicroWalkScratch scr;
            for (size_t t = 0; t < cnt; ++t) {
              const Vec3 p{c[4 * t], c[4 * t + 1], c[4 * t + 2]};
              try {
                ex[t] = expanded ? microwalk_e_transit(s, p, c[4 * t + 3], expansion, n, rngs[t],
                                                       scr, step_cap)
                                 : microwalk_transit_lazy(s, {p, c[4 * t + 3]}, n, rngs[t], scr,
                                                          step_cap);
              } catch (const EngulfedStart&) {
                ex[t].kind = Exit::Kind::Conductor;
                ex[t].conductor_id = -1;
                ex[t].steps = 0;
              }
            }
          } else {
            std::vector<Cube> cb(cnt);
            for (size_t t = 0; t < cnt; ++t)
              cb[t] = {{c[4 * t], c[4 * t + 1], c[4 * t + 2]}, c[4 * t + 3]};
            ex = microwalk_structure_transits(s, cb, n, expanded, rngs, step_cap);
          }
        }
        return exits_dict(ex, rngs);
      },
      py::arg("structure_json"), py::arg("cubes"), py::arg("n"), py::arg("expanded"),
      py::arg("expansion") = 5.0, py::arg("states"), py::arg("single") = false,
      py::arg("step_cap") = 0);

  m.def(
      "neighbor_weights",
      [](py::array_t<double, py::array::c_style | py::array::forcecast> eps,
         std::vector<int> node) {
        DielectricGrid g;
        g.n = static_cast<int>(std::lround(std::cbrt(static_cast<double>(eps.size()))));
        g.cube = {{0, 0, 0}, g.n / 2.0};
        g.eps.assign(eps.data(), eps.data() + eps.size());
        return neighbor_weights(g, {node.at(0), node.at(1), node.at(2)});
      },
      py::arg("eps"), py::arg("node"));

  m.def(
      "build_grid",
      [](const std::string& text, std::vector<double> center, double hw, int n,
         bool allow_conductors) {
        const Structure s = parse_structure(text);
        const DielectricGrid g = build_grid(s, {{center.at(0), center.at(1), center.at(2)}, hw},
                                            n, allow_conductors);
        py::array_t<double> eps(g.eps.size());
        std::copy(g.eps.begin(), g.eps.end(), eps.mutable_data());
        py::object mask = py::none();
        if (g.has_mask()) {
          py::array_t<int32_t> mk(g.conductor_mask.size());
          std::copy(g.conductor_mask.begin(), g.conductor_mask.end(), mk.mutable_data());
          mask = mk;
        }
        return py::make_tuple(eps, mask, static_cast<int>(g.tag), g.strat_axis);
      },
      py::arg("structure_json"), py::arg("center"), py::arg("half_width"), py::arg("n"),
      py::arg("allow_conductors") = false);

  // host direct solves (direct.cpp): the band L D L^T fallback of solve_sgf
  // and oracle.hpp's dense exact_absorption_row -- B200 extras for tests
  auto grid_of = [](py::array_t<double, py::array::c_style | py::array::forcecast> eps,
                    double hw, py::object mask) {
    DielectricGrid g;
    g.n = static_cast<int>(std::lround(std::cbrt(static_cast<double>(eps.size()))));
    g.cube = {{0, 0, 0}, hw > 0 ? hw : g.n / 2.0};
    g.eps.assign(eps.data(), eps.data() + eps.size());
    if (!mask.is_none()) {
      auto mk = py::cast<py::array_t<int32_t, py::array::c_style | py::array::forcecast>>(mask);
      g.conductor_mask.assign(mk.data(), mk.data() + mk.size());
    }
    return g;
  };
  m.def(
      "direct_sgf",
      [grid_of](py::array_t<double, py::array::c_style | py::array::forcecast> eps, double hw,
                py::object mask) {
        const DirectSgf d = direct_sgf(grid_of(eps, hw, mask), true);
        const size_t P = d.sgf.probs.size();
        py::array_t<double> probs(P), ker({static_cast<size_t>(3), P});
        std::copy(d.sgf.probs.begin(), d.sgf.probs.end(), probs.mutable_data());
        for (int a = 0; a < 3; ++a)
          std::copy(d.sgf.grad_kernels[a].begin(), d.sgf.grad_kernels[a].end(),
                    ker.mutable_data() + a * P);
        py::dict o;
        o["probs"] = probs;
        o["kernels"] = ker;
        o["pitch"] = d.sgf.pitch;
        o["expected_steps"] = d.expected_steps;
        return o;
      },
      py::arg("eps"), py::arg("half_width") = 0.0, py::arg("mask") = py::none());
  m.def(
      "exact_absorption_row",
      [grid_of](py::array_t<double, py::array::c_style | py::array::forcecast> eps,
                py::object mask, int cap) {
        const std::vector<double> r = exact_absorption_row(grid_of(eps, 0.0, mask), cap);
        py::array_t<double> out(r.size());
        std::copy(r.begin(), r.end(), out.mutable_data());
        return out;
      },
      py::arg("eps"), py::arg("mask") = py::none(), py::arg("cap") = 12);

  // StratifiedSgfCache (sgf_cache.hpp:47-101) -- B200 extra for tests and tools
  py::class_<StratifiedSgfCache>(m, "SgfCache")
      .def(py::init<size_t>(), py::arg("capacity") = 0)
      .def("get",
           [](StratifiedSgfCache& c, int n, int axis, const std::vector<double>& layers) {
             std::shared_ptr<const DiscreteSGF> g;
             {
               py::gil_scoped_release release;
               g = c.get(profile_key(n, axis, layers));
             }
             return py::array_t<double>(g->probs.size(), g->probs.data());
           },
           py::arg("n"), py::arg("axis"), py::arg("layers"))
      .def("find",
           [](const StratifiedSgfCache& c, int n, int axis,
              const std::vector<double>& layers) -> py::object {
             const auto g = c.find(profile_key(n, axis, layers));
             if (!g) return py::none();
             return py::array_t<double>(g->probs.size(), g->probs.data());
           },
           py::arg("n"), py::arg("axis"), py::arg("layers"))
      .def("kernels",
           [](const StratifiedSgfCache& c, int n, int axis, const std::vector<double>& layers) {
             const auto g = c.find(profile_key(n, axis, layers));
             if (!g || g->grad_kernels[0].empty()) throw py::key_error("no kernels for key");
             const size_t P = g->probs.size();
             py::array_t<double> k({static_cast<size_t>(3), P});
             for (int a = 0; a < 3; ++a)
               std::copy(g->grad_kernels[a].begin(), g->grad_kernels[a].end(),
                         k.mutable_data() + a * P);
             return k;
           })
      .def("stats",
           [](const StratifiedSgfCache& c) {
             const auto st = c.stats();
             py::dict d;
             d["hits"] = st.hits;
             d["misses"] = st.misses;
             d["size"] = st.size;
             return d;
           })
      .def("save", &StratifiedSgfCache::save, py::arg("path"), py::arg("only_n") = 0)
      .def("load", &StratifiedSgfCache::load, py::arg("path"))
      .def("clear", &StratifiedSgfCache::clear);

  m.def("sgf_cache_save", [](const std::string& path) { shared_cache().save(path); });
  m.def("sgf_cache_load", [](const std::string& path) { return shared_cache().load(path); });
  m.def("sgf_cache_clear", []() {
    shared_cache().clear();
    clear_device_tables();  // the device tables mirror the cache: a cleared cache solves anew
  });
  m.def("sgf_cache_stats", []() {
    const auto st = shared_cache().stats();
    py::dict d;
    d["hits"] = st.hits;
    d["misses"] = st.misses;
    d["size"] = st.size;
    return d;
  });

  m.attr("__version__") = "1.0.0";
}
