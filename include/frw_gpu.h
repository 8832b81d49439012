/*
 * frw_gpu.h -- C ABI of the B200-native FRW / MicroWalk hot path
 * (libfrwgpu.so, sm_100a).  Plain C: POD in and out, int status codes,
 * no exceptions, no torch types.  The C++ host layer
 * (paper_2507_09730_b200/csrc/host, the `frwcap` API mirror) and the ctypes
 * tests call these entry points; INTEGRATION.md shows the binding a
 * maintainer of the reference would add.
 *
 * The reference (/root/reference/proj) has no C ABI: its boundary is the C++
 * API in proj/include/frwcap/*.hpp and the pybind11 module _core
 * (bindings/py_module.cpp).  Each entry point below names the reference
 * interface it replaces.
 *
 * Ownership: one context per device; calls on one context are serialized
 * by the caller.  Device buffers are owned by the context; host buffers by
 * the caller.  Functions suffixed _dev take device pointers and run
 * asynchronously on the context stream; the others take host pointers and
 * return after the results are copied back.
 */
#ifndef FRW_GPU_H
#define FRW_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct frw_ctx frw_ctx;

/* Status codes; the C++ host maps them back to the reference exception
 * types (SURVEY.md §8(b) "Error conventions"). */
enum {
  FRW_OK = 0,
  FRW_EINVAL = -1,    /* std::invalid_argument                           */
  FRW_ECUDA = -2,     /* CUDA runtime failure                            */
  FRW_ESTEPCAP = -3,  /* std::runtime_error: step cap exceeded           */
                      /*   (microwalk.cpp:81, :153-155)                  */
  FRW_EENGULFED = -4, /* EngulfedStart (microwalk.hpp:31-33)             */
  FRW_ESOLVE = -5,    /* SolveError (sgf.hpp:104-109)                    */
  FRW_ENOMEM = -6,
  FRW_EMISS = -7      /* stratified-SGF table miss (handled by the host) */
};

/* Random streams.  SPLITMIX_PARITY replays the reference stream of each
 * transit/walk bit for bit (rng.hpp:12-40, SplitMix64(seed, stream));
 * PHILOX is the production generator, Philox4x32-10 keyed by seed with
 * counter (transit or walk id, step). */
/* FRW_RNG_SPLITMIX_PARITY: transit/walk t draws from SplitMix64(seed, t)
 * (rng.hpp:16-17), bit-exact with the reference.  FRW_RNG_PHILOX: Philox4x32-10
 * keyed by seed, counter (t, step block).  FRW_RNG_SPLITMIX_STATES: transit t
 * continues a caller-owned SplitMix64 whose raw state is states[t] (the
 * single-transit API, microwalk.hpp:77-100); the state after the transit is
 * states[t] + steps * 0x9E3779B97F4A7C15. */
enum { FRW_RNG_SPLITMIX_PARITY = 0, FRW_RNG_PHILOX = 1, FRW_RNG_SPLITMIX_STATES = 2 };

/* ---- context ------------------------------------------------------------ */
int frw_ctx_create(int device, frw_ctx **out);
void frw_ctx_destroy(frw_ctx *ctx);
const char *frw_last_error(const frw_ctx *ctx);
/* device properties the bench reports (SM count, clock kHz) */
int frw_device_info(const frw_ctx *ctx, int *sm_count, int *sm_clock_khz,
                    char *name, int name_len);
/* optional: run on an existing cudaStream_t (e.g. torch's current stream) */
int frw_set_stream(frw_ctx *ctx, void *cuda_stream);
int frw_synchronize(frw_ctx *ctx);

/* ---- single transition cube (configs C1/C2) ----------------------------- */
/* Replaces constructing a DielectricGrid (geometry.hpp:151-172) for
 * microwalk_transit(const DielectricGrid&, ...) (microwalk.hpp:77-79).
 * eps: n^3 relative permittivities, x fastest (idx = (k*n+j)*n+i);
 * mask: n^3 conductor ids (-1 free) or NULL.  The cube is centred at
 * (cx,cy,cz) with the given half width.  The upload compiles the grid into
 * the device stencil table (one 16-bit record id per node plus a table of
 * distinct step records). */
int frw_upload_grid(frw_ctx *ctx, int n, const double *eps,
                    const int32_t *mask, double cx, double cy, double cz,
                    double half_width);

/* Host-only compilation of a cube into the stencil table (no device calls;
 * used by the CPU tests to check the threshold construction).  Pass NULL
 * buffers to query *records first; map has (n+2)^3 entries (the lattice
 * with a one-node halo, x-fastest; halo nodes and conductor voxels hold the
 * exit record records-1), rec `records` packed words (five 11-bit threshold
 * lanes 2047 - T_d at bits 12d, guard bits 12d+11), full 5*records exact
 * 53-bit thresholds. */
int frw_grid_compile(int n, const double *eps, const int32_t *mask,
                     uint16_t *map, uint64_t *rec, uint64_t *full,
                     int *records);
/* bytes the last frw_upload_grid copied host->device */
int frw_grid_h2d_bytes(const frw_ctx *ctx, uint64_t *bytes);

/* Upload statistics: distinct step records, bytes staged per CTA in shared
 * memory, whether the table is shared-memory resident. */
int frw_grid_info(const frw_ctx *ctx, int *records, int *smem_bytes,
                  int *smem_resident);

typedef struct {
  int rng_mode;          /* FRW_RNG_*                                     */
  uint64_t seed;
  uint64_t stream_begin; /* transit t uses stream stream_begin + t         */
  int64_t count;         /* number of transits                             */
  int32_t step_cap;      /* 0: 1000*n^2, like microwalk.cpp:81             */
  int32_t blocks;        /* 0: one persistent CTA per SM                   */
  const uint64_t *states; /* FRW_RNG_SPLITMIX_STATES: [count] raw states    */
} frw_mw_params;

/* Outputs.  panels/steps/cond are per transit (may be NULL): panel is the
 * surface panel (surface_panel_of, sgf.cpp:13-30) or -1 for a conductor
 * exit (cond then holds the conductor id).  hist has 6n^2 bins counting
 * surface exits.  step_sum/step_sumsq are exact integer moments of the
 * step count; cond_exits counts conductor exits. */
typedef struct {
  int32_t *panels;
  int32_t *steps;
  int32_t *cond;
  uint64_t *hist;
  uint64_t *step_sum;   /* [1] */
  uint64_t *step_sumsq; /* [1] */
  uint64_t *cond_exits; /* [1] */
  int64_t *exit_nd;     /* per transit: node index * 8 + exit direction
                           (Exit::voxel / Exit::dir, microwalk.hpp:18-27) */
} frw_mw_out;

/* Host-pointer batch: runs `count` transits of the uploaded cube
 * (microwalk_transit, microwalk.cpp:188-197, batched) and copies the
 * requested outputs back.  hist/moments are overwritten, not accumulated. */
int frw_microwalk_batch(frw_ctx *ctx, const frw_mw_params *p,
                        const frw_mw_out *host_out);
/* Device-pointer batch, asynchronous on the context stream.  hist and the
 * moments are ACCUMULATED into (zero them first to overwrite). */
int frw_microwalk_batch_dev(frw_ctx *ctx, const frw_mw_params *p,
                            const frw_mw_out *dev_out);
/* the error flag of the last _dev launch (FRW_OK or FRW_ESTEPCAP);
 * synchronizes the context stream */
int frw_microwalk_check(frw_ctx *ctx);

/* ---- floating-random-walk engine (configs C3-C5) ------------------------- */
/* Replaces frwcap::Structure (geometry.hpp:94-121) on the device.  Boxes are
 * lo.xyz,hi.xyz in nm, in declaration order (dielectrics: later wins,
 * geometry.cpp:47-55; conductors: first hit wins, geometry.cpp:57-62). */
typedef struct {
  int32_t n_cond;
  const int32_t *cond_id;
  const double *cond_box;   /* [n_cond][6] */
  int32_t n_diel;
  const double *diel_box;   /* [n_diel][6] */
  const double *diel_eps;   /* [n_diel]    */
  double background_eps;
  double world[6];
} frw_structure;
int frw_upload_structure(frw_ctx *ctx, const frw_structure *s);

/* Stratified-SGF table (StratifiedSgfCache, sgf_cache.hpp:52-108): one entry
 * per ProfileKey (n, axis, layers rounded to 6 significant digits;
 * sgf_cache.cpp:29-51) holding the canonical unit-pitch solve: probs and
 * inclusive cdf over the 6n^2 surface panels and the three gradient kernels
 * (kernels may be NULL for a probs-only entry). */
int frw_sgf_put(frw_ctx *ctx, int n, int axis, const double *layers,
                double pitch, const double *probs, const double *cdf,
                const double *kernels);
int frw_sgf_count(const frw_ctx *ctx, int *entries);
/* Device miss solver (sgf.cpp:57-290 on the canonical grid of each key,
 * sgf_cache.cpp:78-96): `count` keys of lattice size n, axes[count],
 * layers count x n (rounded).  Writes probs (count x 6n^2, clamped at 0 as
 * in sgf.cpp:255-262) and, if non-NULL, kernels (count x 3 x 6n^2) to host
 * memory; does not insert into the table.  FRW_ESOLVE when a PCG fails to
 * converge or the normalization check fails. */
int frw_sgf_solve(frw_ctx *ctx, int n, int count, const int *axes,
                  const double *layers, double *probs, double *kernels);
int frw_sgf_clear(frw_ctx *ctx);

/* Called by frw_run_walks with the keys the table lacks (deduplicated;
 * layers is count x n, row-major); the host solves the canonical grids (or
 * calls frw_sgf_solve) and frw_sgf_put's each before returning 0.  With a
 * NULL callback frw_run_walks solves the misses on the device itself.  The walks that missed
 * are re-run from their start (their random streams are a pure function of
 * the walk id), so results do not depend on when an entry arrived. */
typedef int (*frw_miss_fn)(void *user, int n, int count, const int *axes,
                           const double *layers);

enum { FRW_MODE_FDM = 0, FRW_MODE_MW = 1, FRW_MODE_MWE = 2,
       FRW_MODE_HYBRID_MW = 3, FRW_MODE_HYBRID_MWE = 4 };

/* Engine parameters (Config, engine.hpp:28-43, plus the derived
 * GaussianSurface of engine.cpp:84-124 and snap distance engine.cpp:186). */
typedef struct {
  int32_t grid_n;
  int32_t mode;           /* FRW_MODE_*                                   */
  double expansion;
  double snap;            /* absolute snap distance, nm                   */
  int64_t hop_cap;
  uint64_t seed;
  int32_t rng_mode;       /* FRW_RNG_*                                    */
  int32_t n_slots;        /* resident walk slots, 0 = default             */
  double gauss_box[6];
  double face_cdf[6];
  double area_m2;
} frw_walk_params;

/* Tallies of one frw_run_walks call (overwritten, not accumulated).  Slot
 * arrays have n_cond+1 entries: conductors in declaration order, ground
 * last (engine.cpp:461-468).  Sums are reduced in a fixed order over walk
 * ids, so they are bit-reproducible run to run and independent of the
 * launch shape. */
typedef struct {
  double *sum;
  double *sumsq;
  uint64_t *landed;
  uint64_t aborted;       /* hop-cap or resample-cap walks, in ground     */
  uint64_t resampled;     /* degenerate Gaussian points redrawn           */
  uint64_t first[4];      /* stratified, shrunk, layered, homogenized     */
  uint64_t sub[4];        /* cached, microwalk, microwalk_e, fdm          */
  uint64_t cache_hits;
  uint64_t cache_misses;  /* distinct keys handed to the miss callback    */
  uint64_t mw_steps;      /* total MicroWalk lattice steps                */
  uint64_t restarts;      /* walks re-run after a table miss              */
  uint64_t mw_general_steps; /* MicroWalk steps next to a cell face        */
  uint64_t mw_cell_changes;  /* MicroWalk moves across a cell face         */
  double mw_ms;           /* device time of the MicroWalk kernel          */
  double total_ms;        /* device time of the whole call                */
  uint64_t mw_jumps;      /* MicroWalk lattice jumps (Philox mode)        */
  uint64_t mw_jump_steps; /* lattice steps the jumps stand for (counted in
                             mw_steps as E[tau]); steps actually taken =
                             mw_steps - mw_jump_steps                      */
  uint64_t mw_dense_hops; /* MicroWalk hops whose cube held more than 64
                             boxes, run on a dense voxel grid             */
} frw_tally;

/* Per-walk outcome (Engine::WalkOut, engine.hpp:157-161, plus the walk's
 * dispatch counts).  branch is the first-transition ladder branch (0-3) or
 * 255 when the resample cap was hit. */
typedef struct {
  double weight;       /* first-transition weight, farads                 */
  uint64_t mw_steps;   /* MicroWalk lattice steps taken                   */
  int32_t slot;        /* terminal: conductor declaration index or ground */
  uint32_t cached;     /* cached (stratified) hops                        */
  uint32_t microwalk;  /* MicroWalk hops                                  */
  uint8_t aborted, branch, resampled, done;
} frw_walk_record;

/* Runs walks [walk_begin, walk_begin+count) of the master conductor whose
 * declaration index is `master` (Engine::run_walk, engine.cpp:352-376,
 * batched).  `records` (host array of `count`, may be NULL) receives the
 * per-walk outcomes in walk order, e.g. for a walk-order fold on the host
 * (engine.cpp:461-468). */
int frw_run_walks(frw_ctx *ctx, const frw_walk_params *p, int32_t master,
                  uint64_t walk_begin, int64_t count, frw_miss_fn miss,
                  void *user, frw_tally *out, frw_walk_record *records);

/* Per-chunk tallies of the last successful frw_run_walks on this context: the
 * call's walks in chunks of *chunk (1024) consecutive walk indices from its
 * walk_begin, per chunk sum[nslots], sumsq[nslots], landed[nslots] (each sum
 * taken in walk order) and stats[12] (aborted, resampled, first-transition
 * branches 0-3, cached hops, MicroWalk hops, MicroWalk steps).  The host fold
 * of engine.cpp:461-468 over reference batches that are multiples of the
 * chunk reads these instead of the per-walk records (192 B per 1024 walks and
 * conductor slot against 32 KB of records).  Any pointer may be NULL; arrays
 * hold *nchunks * nslots (stats: *nchunks * 12) entries. */
int frw_walk_chunk_tallies(frw_ctx *ctx, int64_t *nchunks, int32_t *chunk, double *sum,
                           double *sumsq, uint64_t *landed, uint64_t *stats);

/* ---- multi-GPU: the per-conductor tallies across ranks ---
 * Walks shard as contiguous walk-index ranges of ONE seed (rank g of G runs
 * [g*W/G, (g+1)*W/G), the reference's per-thread chunking, engine.cpp:437-458);
 * geometry and SGF tables are replicated; the only exchange is one
 * all-reduce (sum) of each rank's tally.  frw_run_walks leaves its tally on
 * the device as one f64 vector (sum, sum of squares and landed per slot, the
 * dispatch/abort counters); frw_tally_allreduce sums it over the ranks of
 * `comm` (an ncclComm_t, or NULL for the context's own communicator from
 * frw_nccl_init) with a single ncclAllReduce on the context stream and
 * writes the combined tally into `out` (same fields as frw_run_walks; counts
 * exact).  NCCL is loaded at first use (libnccl.so.2; a copy already loaded
 * by the host process, e.g. torch's, is shared).  No reference counterpart:
 * the reference is single-process. */
int frw_nccl_unique_id(void *id128);  /* ncclGetUniqueId, 128 bytes (rank 0) */
int frw_nccl_init(frw_ctx *ctx, const void *id128, int nranks, int rank);
int frw_nccl_destroy(frw_ctx *ctx);
int frw_tally_allreduce(frw_ctx *ctx, void *comm, frw_tally *out);

/* One lattice transit per entry over a cube of the uploaded structure:
 * microwalk_transit_lazy (microwalk.cpp:199-204; with_conductors = 0) or the
 * expanded-cube transit of microwalk_e_transit (microwalk.cpp:206-228;
 * with_conductors = 1, the caller has already applied min(expansion*h, wall)
 * and transit_cube).  cubes: [count][4] centre xyz, half width (nm); states:
 * [count] raw SplitMix64 states (advanced by steps * gamma).  kind: 0
 * surface exit, 1 conductor exit (conductor = declaration index), -1
 * EngulfedStart (start voxel inside a conductor).  Step-cap overruns fail the
 * call with FRW_ESTEPCAP.  Host buffers; synchronous. */
typedef struct {
  int32_t kind;
  int32_t panel;
  int32_t conductor;
  int32_t dir;
  int32_t voxel[3];
  int32_t steps;
  double point[3];
} frw_exit;
int frw_structure_transits(frw_ctx *ctx, int n, int count, const double *cubes,
                           int with_conductors, const uint64_t *states, int32_t step_cap,
                           frw_exit *out);
/* Production-mode transits of the same cubes: transit t draws from
 * Philox4x32-10 (seed, t); with jumps != 0 uniform-cell stretches are taken
 * as lattice jumps (the law the walk engine uses in FRW_RNG_PHILOX mode;
 * DESIGN.md §4).  Same outputs as frw_structure_transits; `steps` counts a
 * jump as E[tau] of its radius, stochastically rounded. */
/* The lattice-jump law of radius m (2 <= m <= 31; host-only, no context):
 * the simple symmetric walk's first-hit probabilities of one face of the
 * L-inf sphere of radius m from its centre, face[(2m-1)^2] indexed v*(2m-1)+u
 * (each of the six faces carries 1/6), and E[tau] (steps to the hit). */
int frw_lattice_jump_law(int m, double *face, double *esteps);
int frw_structure_transits_philox(frw_ctx *ctx, int n, int count, const double *cubes,
                                  int with_conductors, uint64_t seed, int jumps,
                                  int32_t step_cap, frw_exit *out);

/* Structure queries on the device (geometry.hpp:101-121), for unit parity
 * with the reference on random scenes.  Per point (points [count][3], nm):
 * conductor_at -- Structure::conductor_at(p, tol) (geometry.cpp:57-62) as the
 * conductor's declaration index, -1 for none; free_half_width --
 * max_free_cube(p).half_width (:64-80), -1 where the reference throws
 * (outside the world or inside a conductor); eps -- permittivity_at(p)
 * (:47-55), NaN outside the world; hop_code / hop_half_width -- the walk
 * engine's one-pass transition prologue (engine.cpp:293-298 with snap = tol):
 * conductor index (Terminate), -1 (TerminateGround), -2 (error) or -3 with
 * the free cube's half width.  Host buffers; synchronous. */
int frw_geometry_queries(frw_ctx *ctx, int count, const double *points, double tol,
                         int32_t *conductor_at, double *free_half_width, double *eps,
                         int32_t *hop_code, double *hop_half_width);
/* The stratification probe + profile key of transition cubes
 * (stratified_profile, geometry.cpp:357-396; profile_key,
 * sgf_cache.cpp:29-51): cubes [count][4] centre xyz, half width (the cube
 * must lie in the world, as every transition cube does); axis[count] is the
 * key axis (uniform profiles normalised to 0) or -1 for a general cube;
 * layers [count][n] the 6-significant-digit layers (0 for general cubes). */
int frw_stratified_keys(frw_ctx *ctx, int n, int count, const double *cubes, int32_t *axis,
                        double *layers);

/* Engine::first_transition / Engine::transition (engine.hpp:146-159;
 * engine.cpp:201-350), one per entry, continuing caller-owned SplitMix64
 * states (states[] in/out).  prm selects grid_n, mode, expansion, snap and
 * the Gaussian area/surface as for frw_run_walks (rng_mode and n_slots are
 * ignored).  Table misses are solved on the device (or through `miss`) and
 * the entry re-run, so no entry reports a miss.  Host buffers. */
typedef struct {
  int32_t ok;      /* 1 transition, 0 degenerate free cube (redraw)          */
  int32_t branch;  /* ladder branch 0..3 (DispatchStats order)               */
  double weight;   /* farads                                                 */
  double point[3];
} frw_first;
/* solve_sgf + expected_steps of `count` unmasked materialised grids
 * (assemble_system / solve_sgf / expected_steps, sgf.cpp:57-299): eps
 * [count][n^3] x-fastest, cube half width (sets the kernels' pitch).
 * probs [count][6n^2], kernels [count][3][6n^2], steps [count] (E[tau] at
 * start_node); any output may be NULL.  Jacobi-PCG, tol 1e-10, cap 20 rows. */
int frw_grid_sgf_solve(frw_ctx *ctx, int n, int count, const double *eps,
                       double half_width, double *probs, double *kernels, double *steps);

/* The reference's full-domain finite-volume capacitance solver
 * (reference_capacitance, oracle.cpp:92-213; validation machinery): R^3
 * voxels over the world box, one CG per terminal.  cap: [n_cond][n_cond]
 * row-major farads, cap[i*n + t] = charge on conductor i when t is at 1 V;
 * residual: worst relative CG residual.  16 <= R, R^3 <= 3.5e6. */
int frw_reference_capacitance(frw_ctx *ctx, const frw_structure *s, int resolution,
                              double *cap, double *residual);

int frw_first_transitions(frw_ctx *ctx, const frw_walk_params *prm, int count,
                          const double *gpoints, const int32_t *axis_sign,
                          uint64_t *states, frw_miss_fn miss, void *user,
                          frw_first *out);

typedef struct {
  int32_t kind;      /* 0 continue, 1 terminate on a conductor, 2 ground    */
  int32_t conductor; /* declaration index (kind 1)                          */
  int32_t dispatch;  /* -1 snapped, 0 cached, 1 microwalk, 2 microwalk_e, 3 fdm */
  int32_t pad;
  double point[3];   /* continue: next point                                */
  uint64_t mw_steps; /* lattice steps of a MicroWalk transition             */
} frw_event;
int frw_transitions(frw_ctx *ctx, const frw_walk_params *prm, int count,
                    const double *points, uint64_t *states, frw_miss_fn miss,
                    void *user, frw_event *out);

/* Events on the context stream for device timing of _dev launches:
 * elapsed ms between frw_event_record(ctx, 0) and frw_event_record(ctx, 1). */
int frw_event_record(frw_ctx *ctx, int which);
int frw_event_elapsed_ms(frw_ctx *ctx, float *ms);

/* Device memory helpers for callers without their own allocator. */
int frw_dev_alloc(frw_ctx *ctx, size_t bytes, void **ptr);
int frw_dev_free(frw_ctx *ctx, void *ptr);
int frw_dev_memset(frw_ctx *ctx, void *ptr, int value, size_t bytes);
/* Page-locked host memory (fast copies of per-walk records / outputs). */
int frw_host_alloc(frw_ctx *ctx, size_t bytes, void **ptr);
int frw_host_free(frw_ctx *ctx, void *ptr);
int frw_memcpy_h2d(frw_ctx *ctx, void *dst, const void *src, size_t bytes);
int frw_memcpy_d2h(frw_ctx *ctx, void *dst, const void *src, size_t bytes);

/* Shared-memory bandwidth probe used as the on-chip roofline denominator:
 * every SM streams `iters` 128-bit conflict-free LDS per thread; returns
 * bytes/s measured with device events. */
int frw_smem_bandwidth_probe(frw_ctx *ctx, int iters, double *bytes_per_s);

#ifdef __cplusplus
}
#endif
#endif /* FRW_GPU_H */
