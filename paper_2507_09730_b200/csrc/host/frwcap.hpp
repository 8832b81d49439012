// frwcap.hpp -- host C++ API of the B200 build, mirroring the reference's
// public solver API (proj/include/frwcap/{geometry,engine,sgf,sgf_cache,
// microwalk}.hpp) so callers switch by relinking.  Everything that walks
// runs on the device through the C ABI in include/frw_gpu.h; this layer
// owns parsing, validation, the SGF cache (miss solves), the batch /
// convergence loop and the result bookkeeping.
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <iosfwd>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

#include "frw_gpu.h"

namespace frwcap {

inline constexpr double kEps0 = 8.8541878128e-12;  // F/m (constants.hpp:5)
inline constexpr double kMetersPerNm = 1e-9;       // constants.hpp:6

// ---- geometry (geometry.hpp:14-121) ---------------------------------------
struct Vec3 {
  double x = 0, y = 0, z = 0;
  double operator[](int a) const { return a == 0 ? x : (a == 1 ? y : z); }
  double& operator[](int a) { return a == 0 ? x : (a == 1 ? y : z); }
  Vec3 operator+(const Vec3& o) const { return {x + o.x, y + o.y, z + o.z}; }
  Vec3 operator-(const Vec3& o) const { return {x - o.x, y - o.y, z - o.z}; }
  bool operator==(const Vec3& o) const = default;
};

struct Vec3i {
  int x = 0, y = 0, z = 0;
  int operator[](int a) const { return a == 0 ? x : (a == 1 ? y : z); }
  int& operator[](int a) { return a == 0 ? x : (a == 1 ? y : z); }
  bool operator==(const Vec3i& o) const = default;
};

struct Box {
  Vec3 lo, hi;
  bool contains(const Vec3& p) const;
  double chebyshev_to(const Vec3& p) const;
  double chebyshev_to_wall(const Vec3& p) const;
  bool contains_box(const Box& o) const;
  bool valid() const;
  // open-interval overlap: touching faces do not count (geometry.hpp:49-52)
  bool intersects_open(const Box& o) const {
    return lo.x < o.hi.x && o.lo.x < hi.x && lo.y < o.hi.y && o.lo.y < hi.y && lo.z < o.hi.z &&
           o.lo.z < hi.z;
  }
  Vec3 center() const { return {(lo.x + hi.x) / 2, (lo.y + hi.y) / 2, (lo.z + hi.z) / 2}; }
  Vec3 half_extent() const { return {(hi.x - lo.x) / 2, (hi.y - lo.y) / 2, (hi.z - lo.z) / 2}; }
};

struct Conductor {
  int id = 0;
  Box box;
};
struct Dielectric {
  Box box;
  double eps_r = 1.0;
};

class ParseError : public std::runtime_error {
 public:
  ParseError(int line, int column, const std::string& what)
      : std::runtime_error("parse error at line " + std::to_string(line) + ", column " +
                           std::to_string(column) + ": " + what),
        line(line),
        column(column) {}
  int line, column;
};
class ValidationError : public std::runtime_error {
  using std::runtime_error::runtime_error;
};

// result of the conductor-free cube query (geometry.hpp:93-97)
struct FreeCube {
  double half_width = 0;
  std::optional<int> nearest_id;  // empty when the world wall is nearest
};

struct Structure {
  std::vector<Conductor> conductors;
  std::vector<Dielectric> dielectrics;
  double background_eps = 1.0;
  Box world;
  int master_id = 0;

  double permittivity_at(const Vec3& p) const;
  std::optional<int> conductor_at(const Vec3& p, double tol) const;
  FreeCube max_free_cube(const Vec3& p) const;
  const Conductor* find_conductor(int id) const;
  void validate() const;
};

Structure parse_structure(std::string_view text, double world_margin = 5.0);
Structure parse_structure_file(const std::string& path, double world_margin = 5.0);

// permittivity comparison at relative tolerance 1e-9 (geometry.cpp:17-19)
bool eps_equal(double a, double b);

// ---- transition-cube voxelisation (geometry.hpp:124-182) --------------------
enum class GridTag : uint8_t { Uniform, Stratified, General };

struct Cube {
  Vec3 center;
  double half_width = 0;
  Box box() const {
    return {{center.x - half_width, center.y - half_width, center.z - half_width},
            {center.x + half_width, center.y + half_width, center.z + half_width}};
  }
};

// N^3 permittivity lattice of one cube, x-fastest; conductor_mask (-1 free,
// else the conductor id) only when built with allow_conductors
struct DielectricGrid {
  int n = 0;
  Cube cube;
  std::vector<double> eps;
  std::vector<int32_t> conductor_mask;
  GridTag tag = GridTag::Uniform;
  int strat_axis = -1;
  int index(int i, int j, int k) const { return (k * n + j) * n + i; }
  double eps_at(int i, int j, int k) const { return eps[index(i, j, k)]; }
  bool has_mask() const { return !conductor_mask.empty(); }
  int conductor(int i, int j, int k) const {
    return has_mask() ? conductor_mask[index(i, j, k)] : -1;
  }
  double pitch() const { return 2.0 * cube.half_width / n; }
  Vec3 voxel_center(int i, int j, int k) const {
    const double h = cube.half_width, p = pitch();
    return {cube.center.x - h + (i + 0.5) * p, cube.center.y - h + (j + 0.5) * p,
            cube.center.z - h + (k + 0.5) * p};
  }
};
void classify_grid(DielectricGrid& g);
DielectricGrid build_grid(const Structure& s, const Cube& cube, int n,
                          bool allow_conductors = false);

// stratification probe of a cube (geometry.hpp:184-196): the permittivity
// depends on `axis` only; layers[t] at the centre of slice t
struct StratifiedProfile {
  int axis = 0;
  std::vector<double> layers;
  bool uniform() const;  // every layer eps_equal to the first
};
std::optional<StratifiedProfile> stratified_profile(const Structure& s, const Cube& cube, int n);

// ---- lattice and panel algebra (sgf.hpp:24-61, sgf.cpp:13-55) ---------------
inline constexpr int kDirAxis[6] = {0, 0, 1, 1, 2, 2};
inline constexpr int kDirSign[6] = {-1, +1, -1, +1, -1, +1};
inline int surface_panel_index(int n, int face, int u, int v) { return (face * n + v) * n + u; }
int surface_panel_of(int n, const Vec3i& voxel, int dir);
std::array<int, 3> decode_surface_panel(int n, int panel);
Vec3 surface_panel_center(const Cube& cube, int n, int panel);
std::array<double, 2> surface_panel_offsets(int n, int panel);
inline Vec3i start_node(int n) {
  const int c = (n - 1) / 2;
  return {c, c, c};
}
// the walk lattice placed so the point sits on start_node(n)
// (microwalk.hpp:39-44)
inline Cube transit_cube(const Vec3& p, double half_width, int n) {
  if (n % 2 == 1) return {p, half_width};
  const double delta = half_width / (n + 1);
  const double h = (half_width - delta) * (1.0 - 1e-12);
  return {{p.x + delta, p.y + delta, p.z + delta}, h};
}

// ---- SplitMix64 streams (rng.hpp:12-40) ---------------------------------------
class SplitMix64 {
 public:
  SplitMix64() = default;
  explicit SplitMix64(uint64_t seed) : state_(mix(seed)) {}
  SplitMix64(uint64_t seed, uint64_t stream) : state_(mix(mix(seed) + (stream + 1) * kGamma)) {}
  uint64_t next() {
    state_ += kGamma;
    return mix(state_);
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  uint64_t below(uint64_t n) { return next() % n; }
  static uint64_t mix(uint64_t z) {
    z += kGamma;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  // B200: the raw state crosses to the device (FRW_RNG_SPLITMIX_STATES)
  uint64_t state() const { return state_; }
  void set_state(uint64_t s) { state_ = s; }
  void skip(uint64_t draws) { state_ += draws * kGamma; }
  static constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;

 private:
  uint64_t state_ = 0;
};

// Per-caller state of the reference (memo arrays); here it only selects the
// device, the transits themselves keep no host-side memo.
class MicroWalkScratch {
 public:
  void prepare(int n_) {
    n = n_;
    ++epoch;
  }
  int n = 0;
  bool memoize = true;
  uint64_t epoch = 0;
  int device = 0;
};

// ---- SGF (sgf.hpp:116-147) and its cache (sgf_cache.hpp) -------------------
struct DiscreteSGF {
  int n = 0;
  double pitch = 1.0;
  std::vector<double> probs, cdf;
  std::array<std::vector<double>, 3> grad_kernels;
  bool has_kernels() const { return !grad_kernels[0].empty(); }
};

class SolveError : public std::runtime_error {
 public:
  SolveError(const std::string& what, double residual)
      : std::runtime_error(what), residual(residual) {}
  double residual = 0;
};

double round_sig(double x, int digits);

// sgf_cache.hpp:20-48: the identity of a solved canonical SGF.  `expanded`
// and `conductor_sig` key MicroWalk-E / masked-grid solves; the walk engine's
// device table holds the plain stratified keys only.
struct ProfileKey {
  int n = 0;
  int axis = 0;
  std::vector<double> layers;  // rounded to 6 significant digits
  bool expanded = false;
  std::optional<uint64_t> conductor_sig;
  bool operator==(const ProfileKey&) const = default;
};
struct ProfileKeyHash {
  size_t operator()(const ProfileKey& k) const;
};
ProfileKey profile_key(int n, int axis, const std::vector<double>& layers, bool expanded = false,
                       std::optional<uint64_t> conductor_sig = {});
ProfileKey profile_key(const StratifiedProfile& profile, int n);
// from a materialised Uniform or Stratified grid; throws on General
ProfileKey profile_key(const DielectricGrid& grid);
// order-sensitive hash of a grid's conductor mask, for keys of masked grids
uint64_t conductor_signature(const DielectricGrid& grid);

// unit-pitch grid of a key's layers; throws for conductor-signature keys
DielectricGrid canonical_grid(const ProfileKey& key);
// canonical unit-pitch solve of a key (sgf_cache.cpp:78-131 + sgf.cpp:231-290)
DiscreteSGF solve_canonical(const ProfileKey& key, bool with_kernels = true, int device = 0);

class StratifiedSgfCache {
 public:
  explicit StratifiedSgfCache(size_t capacity = 0) : capacity_(capacity) {}
  void set_device(int device) { device_ = device; }
  std::shared_ptr<const DiscreteSGF> get(const ProfileKey& key);
  // a miss solves the caller's (Uniform or Stratified) grid instead
  std::shared_ptr<const DiscreteSGF> get(const ProfileKey& key,
                                         const std::function<DielectricGrid()>& provider);
  std::shared_ptr<const DiscreteSGF> find(const ProfileKey& key) const;
  // solves the missing keys (one device batch per lattice size)
  void solve_many(const std::vector<ProfileKey>& keys, int threads = 0);
  // first stored result wins (sgf_cache.cpp:133-153)
  std::shared_ptr<const DiscreteSGF> insert(const ProfileKey& key,
                                            std::shared_ptr<const DiscreteSGF> sgf);
  void count_misses(uint64_t k);
  struct Stats {
    uint64_t hits = 0, misses = 0;
    size_t size = 0;
  };
  Stats stats() const;
  void clear();
  std::vector<std::pair<ProfileKey, std::shared_ptr<const DiscreteSGF>>> entries() const;
  // SGF1 persistence (sgf_cache.cpp:210-324)
  void save(const std::string& path, int only_n = 0) const;
  size_t load(const std::string& path);

 private:
  // capacity > 0: least-recently-used entries (last get/find/store) are
  // evicted on insert (sgf_cache.hpp:51-55, sgf_cache.cpp:133-153)
  struct Entry {
    std::shared_ptr<const DiscreteSGF> sgf;
    mutable uint64_t used = 0;
  };
  std::shared_ptr<const DiscreteSGF> store_locked(const ProfileKey& key,
                                                  std::shared_ptr<const DiscreteSGF> sgf);
  void touch(const Entry& e) const { e.used = ++clock_; }
  size_t capacity_;
  int device_ = 0;
  mutable std::mutex mu_;
  std::unordered_map<ProfileKey, Entry, ProfileKeyHash> map_;
  mutable uint64_t clock_ = 0;
  uint64_t hits_ = 0, misses_ = 0;
};

// ---- engine (engine.hpp:23-177) ---------------------------------------------
enum class Mode { FDM, MW, MWE, HybridMW, HybridMWE };
Mode parse_mode(const std::string& name);
std::string mode_name(Mode mode);

enum class RngMode { SplitMixParity, Philox };

struct Config {
  int grid_n = 24;
  double expansion = 5.0;
  Mode mode = Mode::HybridMWE;
  double rel_std_tol = 0.01;
  long min_walks = 4096;
  long max_walks = 4000000;
  int batch = 1024;
  uint64_t seed = 1;
  double snap_tol = 1e-4;
  long hop_cap = 10000;
  double gaussian_gap_fraction = 0.5;
  double world_margin = 5.0;
  // B200 knobs (defaults keep the reference behaviour)
  RngMode rng = RngMode::Philox;
  bool all_couplings_rule = false;  // stop when every coupling meets tol (C4)
  // walks per frw_run_walks call (each drains its pool through one tail);
  // 0 = auto: up to 2^24 when the walk count is fixed (min == max walks),
  // 2^22 while a stopping rule is tested (a speculative chunk is discarded)
  long device_batch = 0;
  int device = 0;
  // Several devices (one host thread and one context each): device chunks
  // of one walk sequence go round-robin to them and are folded in walk
  // order, so the result equals the one-device run bit for bit
  // (SURVEY.md §8(e)).  Empty: {device}.  A device listed twice gets two
  // contexts (independent streams on one GPU).
  std::vector<int> devices;

  void validate() const;
};

struct GaussianSurface {
  Box box;
  double area_m2 = 0;
  std::array<double, 6> face_cdf{};
};
GaussianSurface gaussian_surface(const Structure& s, double gap_fraction);

struct GaussianSample {
  Vec3 point;
  int axis = 0;  // outward normal axis of the sampled face
  int sign = 1;  // outward normal sign
};
GaussianSample sample_gaussian(const GaussianSurface& g, SplitMix64& rng);

struct WalkEvent {
  enum class Kind { Continue, Terminate, TerminateGround };
  Kind kind = Kind::TerminateGround;
  Vec3 point;             // Continue: next point on the transition cube surface
  int conductor_id = -1;  // Terminate
};

struct FirstTransition {
  Vec3 point;
  double weight = 0;  // farads
  int branch = 0;     // ladder branch taken, DispatchStats order
};

struct DispatchStats {
  uint64_t first_stratified = 0, first_shrunk = 0, first_layered = 0, first_homogenized = 0;
  uint64_t cached = 0, microwalk = 0, microwalk_e = 0, fdm = 0;
  uint64_t first_total() const {
    return first_stratified + first_shrunk + first_layered + first_homogenized;
  }
  uint64_t subsequent_total() const { return cached + microwalk + microwalk_e + fdm; }
  DispatchStats& operator+=(const DispatchStats& o);
};

struct TerminalEstimate {
  int conductor_id = -1;
  double value = 0;
  double std_err = 0;
  uint64_t walks_landed = 0;
};

struct CapacitanceResult {
  int master_id = 0;
  std::vector<TerminalEstimate> terminals;
  uint64_t walks = 0;
  bool converged = false;
  uint64_t aborted = 0;
  uint64_t resampled = 0;
  DispatchStats dispatch;
  uint64_t cache_hits = 0;
  uint64_t cache_misses = 0;
  double t_mw_seconds = 0;
  double t_total_seconds = 0;
  uint64_t mw_steps = 0;       // B200 extra: total lattice steps
  uint64_t mw_jumps = 0;       // B200 extra: lattice jumps (Philox mode)
  uint64_t mw_jump_steps = 0;  // B200 extra: steps the jumps stand for (E[tau], in mw_steps)
  uint64_t mw_dense_hops = 0;  // B200 extra: hops on a dense grid (> 64 boxes in the cube)
  double t_device_seconds = 0; // B200 extra: device time of the walk launches
  const TerminalEstimate* find_terminal(int conductor_id) const;
  const TerminalEstimate& self() const;
};

// Tallies of one walk range (frw_tally): per slot (conductors in
// declaration order, ground last) sum, sum of squares and landed count, plus
// the dispatch counters -- the unit the multi-process path all-reduces.
struct WalkTally {
  std::vector<double> sum, sumsq;
  std::vector<uint64_t> landed;
  uint64_t walks = 0, aborted = 0, resampled = 0, mw_steps = 0, mw_jumps = 0, mw_jump_steps = 0,
           mw_dense_hops = 0;
  uint64_t first[4] = {0, 0, 0, 0};  // DispatchStats order
  uint64_t sub[4] = {0, 0, 0, 0};    // cached, microwalk, microwalk_e, fdm
  double mw_ms = 0, total_ms = 0;
};

// Shared device context (one per device and process).
class Device {
 public:
  // `instance` > 0 opens further contexts on the same device
  static Device& get(int device, int instance = 0);
  frw_ctx* ctx() const { return ctx_; }
  ~Device();

 private:
  explicit Device(int device);
  frw_ctx* ctx_ = nullptr;
};

void throw_status(frw_ctx* ctx, int rc);
// drops every stratified-SGF entry the engines put on the devices (they are
// re-put from the host cache on the next call)
void clear_device_tables();

class Engine {
 public:
  Engine(const Structure& s, const Config& cfg, StratifiedSgfCache* cache = nullptr);
  const GaussianSurface& surface() const { return surface_; }
  double snap_distance() const { return snap_; }
  StratifiedSgfCache& cache() { return *cache_; }
  CapacitanceResult extract(int threads = 0);
  // per-walk outcomes of walks [begin, begin+count) (parity tests)
  std::vector<frw_walk_record> run_walks(uint64_t begin, int64_t count);
  // device tallies of walks [begin, begin+count) of the seed's one walk
  // sequence (a rank's share); with `allreduce` they are
  // summed over the ranks of the context's NCCL communicator
  // (frw_nccl_init) by frw_tally_allreduce before they are returned
  WalkTally run_tally(uint64_t begin, int64_t count, bool allreduce = false);
  frw_ctx* context() const { return ctx_; }

  // One weighted first transition / one subsequent transition on the device,
  // continuing the caller's SplitMix64 (engine.hpp:146-159).  Table misses
  // are solved and inserted before the draw, like extract does.
  std::optional<FirstTransition> first_transition(const GaussianSample& g, SplitMix64& rng,
                                                  DispatchStats& stats) const;
  WalkEvent transition(const Vec3& point, SplitMix64& rng, MicroWalkScratch& scratch,
                       DispatchStats& stats, double* t_mw = nullptr) const;
  // batched forms (B200): entry t continues rngs[t]
  std::vector<std::optional<FirstTransition>> first_transitions(
      const std::vector<GaussianSample>& g, std::vector<SplitMix64>& rngs,
      DispatchStats& stats) const;
  std::vector<WalkEvent> transitions(const std::vector<Vec3>& points,
                                     std::vector<SplitMix64>& rngs, DispatchStats& stats) const;

 private:
  void upload() const { upload(ctx_); }
  void upload(frw_ctx* ctx) const;
  frw_walk_params params() const;
  const Structure& s_;
  Config cfg_;
  std::unique_ptr<StratifiedSgfCache> owned_cache_;
  StratifiedSgfCache* cache_;
  GaussianSurface surface_;
  double snap_ = 0;
  int master_slot_ = 0;
  frw_ctx* ctx_ = nullptr;         // first context (single-transition API)
  std::vector<frw_ctx*> ctxs_;     // one per Config::devices entry
};

CapacitanceResult extract(const Structure& s, const Config& cfg, int threads = 0,
                          StratifiedSgfCache* cache = nullptr);

// ---- surface Green's function of a materialised (unmasked) grid, on the device
// (assemble_system + solve_sgf + expected_steps, sgf.cpp:57-299)
// general grids solve on the device (Jacobi-PCG); masked grids, and grids
// whose PCG does not converge, take the host direct solve below (sgf.cpp:162-211)
DiscreteSGF solve_sgf(const DielectricGrid& g, bool with_kernels = true, int device = 0);
double expected_steps(const DielectricGrid& g, int device = 0);

// host direct solve of the transition-cube system (band L D L^T of s_ii,
// direct.cpp): the SGF (surface then conductor panels) and E[steps]; n <= 32
struct DirectSgf {
  DiscreteSGF sgf;
  double expected_steps = 0;
};
DirectSgf direct_sgf(const DielectricGrid& g, bool with_kernels = true);
// oracle.hpp:14-19: the start node's row of a_ii^-1 a_ib by a dense LU
std::vector<double> exact_absorption_row(const DielectricGrid& grid, int cap = 12);
// FD system of a materialised grid (sgf.hpp:75-101).  The B200 build
// assembles s_ii matrix-free on the device, so the system is the grid it is
// built from; solve_sgf / expected_steps of it run the device solver.
struct FDSystem {
  DielectricGrid grid;
  int n = 0;
};
FDSystem assemble_system(const DielectricGrid& g);
DiscreteSGF solve_sgf(const FDSystem& sys, bool with_kernels = true);
double expected_steps(const FDSystem& sys);

// Empirical-vs-exact comparison (oracle.hpp:38-52; validation machinery on
// the host): total variation plus a chi-square statistic over bins pooled to
// an expected count >= 5 (an undersized tail joins the previous group),
// against the Wilson-Hilferty critical value at p = 1e-3.
struct DistributionReport {
  std::vector<double> exact;
  std::vector<double> empirical;
  double tv_distance = 0;
  double gof_statistic = 0;
  double gof_critical = 0;
  int pooled_bins = 0;
  long samples = 0;
  bool gof_pass() const { return gof_statistic <= gof_critical; }
};
DistributionReport compare_distribution(const std::vector<double>& exact,
                                        const std::function<int(SplitMix64&)>& sampler,
                                        long n_samples, SplitMix64& rng);
// oracle.cpp:300-339 test lattices: exponential(mean 10) permittivities
DielectricGrid random_voxel_grid(int n, SplitMix64& rng);
DielectricGrid random_block_grid(int n, int blocks, SplitMix64& rng);

// the reference CLI (cli.cpp:545-620): extract, validate-sgf, bench-scaling,
// oracle-compare; JSON report on `out`, summary on `err`; exit codes 0/1/2
int run_cli(const std::vector<std::string>& args, std::ostream& out, std::ostream& err);

// ---- full-domain FV reference (oracle.hpp:25-31), on the device ----------------
struct ReferenceSolution {
  int resolution = 0;
  std::vector<int> terminal_ids;    // structure declaration order
  std::vector<double> capacitance;  // [n][n] row-major, farads; column t = excitation of t
  double residual = 0;              // worst relative CG residual
  double at(int i, int t) const { return capacitance[i * terminal_ids.size() + t]; }
};
ReferenceSolution reference_capacitance(const Structure& s, int resolution, int device = 0);

// ---- MicroWalk transits (microwalk.hpp:18-100) -------------------------------
struct Exit {
  enum class Kind : uint8_t { Surface, Conductor };
  Kind kind = Kind::Surface;
  int panel = -1;
  int conductor_id = -1;
  Vec3 point;
  Vec3i voxel;
  int dir = -1;
  int steps = 0;
};

class EngulfedStart : public std::runtime_error {
  using std::runtime_error::runtime_error;
};

// beta_i = alpha_i / sum(alpha) at an interior node (microwalk.cpp:160-186)
std::array<double, 6> neighbor_weights(const DielectricGrid& grid, const Vec3i& node);

// One transit per call, on the device, continuing the caller's SplitMix64
// (bit-identical to the reference for the same stream).  Batched forms
// below run many transits per launch.
Exit microwalk_transit(const DielectricGrid& grid, SplitMix64& rng, MicroWalkScratch& scratch,
                       int step_cap = 0);
Exit microwalk_transit(const DielectricGrid& grid, SplitMix64& rng);
Exit microwalk_e_transit(const Structure& s, const Vec3& center, double base_half_width,
                         double expansion, int n, SplitMix64& rng, MicroWalkScratch& scratch,
                         int step_cap = 0);
Exit microwalk_e_transit(const Structure& s, const Vec3& center, double base_half_width,
                         double expansion, int n, SplitMix64& rng);
Exit microwalk_transit_lazy(const Structure& s, const Cube& cube, int n, SplitMix64& rng,
                            MicroWalkScratch& scratch, int step_cap = 0);

// B200 batched forms: transit t continues rngs[t] (advanced in place).
std::vector<Exit> microwalk_transits(const DielectricGrid& grid, std::vector<SplitMix64>& rngs,
                                     int step_cap = 0, int device = 0);
// lazy (with_conductors = false, cubes as given) or expanded (true; cubes
// already min(expansion*h, wall)-sized and transit_cube-placed); a start
// voxel inside a conductor yields kind Conductor with conductor_id -1 and
// steps 0 (EngulfedStart in the single-transit form)
std::vector<Exit> microwalk_structure_transits(const Structure& s, const std::vector<Cube>& cubes,
                                               int n, bool with_conductors,
                                               std::vector<SplitMix64>& rngs, int step_cap = 0,
                                               int device = 0);

// uploads `s` to the context unless it is the structure uploaded last
void upload_structure(frw_ctx* ctx, const Structure& s);

struct TransitBatch {
  std::vector<uint64_t> hist;
  std::vector<int32_t> panels, steps;
  uint64_t step_sum = 0, step_sumsq = 0;
};
TransitBatch microwalk_transit_batch(int n, const std::vector<double>& eps, const Vec3& center,
                                     double half_width, uint64_t seed, uint64_t stream_begin,
                                     int64_t count, RngMode rng, bool per_transit,
                                     int device = 0);

}  // namespace frwcap
