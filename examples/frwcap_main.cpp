// frwcap_main.cpp -- a C++ caller of the B200 build through the reference's
// own C++ API (proj/include/frwcap/*.hpp signatures, csrc/host/frwcap.hpp):
// what an application linked against the reference's libfrwcap looks like
// after relinking against paper_2507_09730_b200/lib/libfrwcap.so.
//
//   frwcap_main extract <structure.json> [walks]    capacitance row (JSON-ish)
//   frwcap_main transit <n> <seed> <count>          microwalk_transit on a
//                                                   random voxel grid
//   frwcap_main cli <args...>                       the reference CLI (run_cli)
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <string>
#include <vector>

#include "frwcap.hpp"

int main(int argc, char** argv) {
  using namespace frwcap;
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s extract|transit|cli ...\n", argv[0]);
    return 2;
  }
  const std::string cmd = argv[1];
  try {
    if (cmd == "extract" && argc >= 3) {
      const Structure s = parse_structure_file(argv[2]);
      Config cfg;
      cfg.mode = Mode::HybridMW;
      cfg.rng = RngMode::SplitMixParity;
      cfg.min_walks = cfg.max_walks = argc >= 4 ? std::atol(argv[3]) : 100000;
      StratifiedSgfCache cache;
      const CapacitanceResult r = extract(s, cfg, 0, &cache);
      std::printf("master %d walks %llu converged %d\n", r.master_id,
                  static_cast<unsigned long long>(r.walks), r.converged ? 1 : 0);
      for (const TerminalEstimate& t : r.terminals)
        std::printf("C %d %.17g %.17g %llu\n", t.conductor_id, t.value, t.std_err,
                    static_cast<unsigned long long>(t.walks_landed));
      return 0;
    }
    if (cmd == "transit" && argc >= 5) {
      const int n = std::atoi(argv[2]);
      SplitMix64 grid_rng(std::strtoull(argv[3], nullptr, 10), 0);
      const DielectricGrid grid = random_voxel_grid(n, grid_rng);
      MicroWalkScratch scratch;
      const long count = std::atol(argv[4]);
      for (long t = 0; t < count; ++t) {
        SplitMix64 rng(7, static_cast<uint64_t>(t));
        const Exit e = microwalk_transit(grid, rng, scratch);
        std::printf("%d %d\n", e.panel, e.steps);
      }
      return 0;
    }
    if (cmd == "cli") {
      std::vector<std::string> args(argv + 2, argv + argc);
      return run_cli(args, std::cout, std::cerr);
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
  std::fprintf(stderr, "bad arguments\n");
  return 2;
}
