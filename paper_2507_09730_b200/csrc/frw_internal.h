// frw_internal.h -- context state shared by the libfrwgpu.so translation
// units (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "frw_gpu.h"

namespace frw {

// Compiled single-cube stencil table (see mw_grid.cu).
struct GridTable {
  int n = 0;
  int records = 0;
  int start_idx = 0;
  bool start_is_conductor = false;
  double center[3] = {0, 0, 0};
  double half_width = 0;
  uint16_t* d_map = nullptr;      // [n^3] node -> record
  uint64_t* d_rec = nullptr;      // [R] packed SWAR record
  uint64_t* d_full = nullptr;     // [R][5] exact 53-bit thresholds
  uint64_t h2d_bytes = 0;         // bytes copied by the last upload
  int32_t* d_mask = nullptr;      // [n^3] conductor ids (valid when has_mask)
  int32_t* d_exit = nullptr;      // [(n+2)^3] absorbing node -> panel, or -2 - conductor id
  bool has_mask = false;
  size_t map_bytes = 0, rec_bytes = 0;  // padded to 16 B
  // allocation capacities (re-uploads of a same-sized grid reuse them)
  size_t blob_cap = 0, full_cap = 0, mask_cap = 0, exit_cap = 0;
  // on-device compile (mw_grid.cu, compile_grid_device): eps staging, the
  // palette / stencil hash tables and counters, one allocation
  char* d_dc = nullptr;
  size_t dc_cap = 0;
  int exit_n = 0;  // exit_info cached for this n (unmasked grids)
  bool host_compiled = false;  // FRW_GRID_HOST_COMPILE / fallback: the last upload compiled on the host
};

}  // namespace frw

struct frw_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::string err;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  int sm_count = 0;
  int sm_clock_khz = 0;
  int max_smem_optin = 0;
  char name[256] = {0};

  frw::GridTable grid;

  // scratch for launches
  unsigned long long* d_ctr = nullptr;  // transit counter
  int* d_err = nullptr;                 // error flag
  // walk engine state (walk.cu); freed through walk_free
  void* walk = nullptr;
  void (*walk_free)(frw_ctx*) = nullptr;

  // host-batch staging
  uint64_t* d_hist = nullptr;
  size_t hist_cap = 0;
  uint64_t* d_mom = nullptr;            // [3]
  int32_t* d_tr = nullptr;              // per-transit outputs and states
  size_t tr_cap = 0;                    // bytes
  // stratified-key solver scratch (sgf_solve.cu), grown on demand
  char* d_solve = nullptr;
  size_t solve_cap = 0;                 // bytes
};

#define FRW_CUDA(ctx, call)                                         \
  do {                                                              \
    cudaError_t e_ = (call);                                        \
    if (e_ != cudaSuccess) {                                        \
      (ctx)->err = std::string(#call) + ": " + cudaGetErrorString(e_); \
      return FRW_ECUDA;                                             \
    }                                                               \
  } while (0)

int frw_fail(frw_ctx* ctx, int code, const std::string& msg);
