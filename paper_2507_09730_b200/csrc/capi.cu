// capi.cu -- context management and device helpers of the C ABI
// (include/frw_gpu.h).
#include <cuda_runtime.h>

#include <cstring>
#include <new>

#include "frw_internal.h"

int frw_fail(frw_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

namespace {
// a probe kernel for the on-chip roofline: conflict-free 128-bit LDS
__global__ void __launch_bounds__(1024) smem_probe_kernel(int iters,
                                                          uint32_t* sink) {
  __shared__ uint4 buf[1024];
  buf[threadIdx.x] = make_uint4(threadIdx.x, 1, 2, 3);
  __syncthreads();
  uint4 acc = make_uint4(0, 0, 0, 0);
  uint32_t off = threadIdx.x;
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint4 v = buf[(off + u * 32) & 1023];
      acc.x ^= v.x;
      acc.y += v.y;
      acc.z ^= v.z;
      acc.w += v.w;
    }
    off += acc.x & 1;  // keep the loop data-dependent
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0xFFFFFFFFu) sink[0] = acc.x;
}
}  // namespace

extern "C" {

int frw_ctx_create(int device, frw_ctx** out) {
  if (!out) return FRW_EINVAL;
  *out = nullptr;
  frw_ctx* ctx = new (std::nothrow) frw_ctx;
  if (!ctx) return FRW_ENOMEM;
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev[0]);
  if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev[1]);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_ctr, sizeof(unsigned long long) * 4);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_err, sizeof(int) * 4);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_mom, sizeof(uint64_t) * 4);
  cudaDeviceProp prop;
  if (e == cudaSuccess) e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) {
    delete ctx;
    return FRW_ECUDA;
  }
  ctx->own_stream = true;
  ctx->sm_count = prop.multiProcessorCount;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, device);
  ctx->sm_clock_khz = clk;
  ctx->max_smem_optin = static_cast<int>(prop.sharedMemPerBlockOptin);
  std::strncpy(ctx->name, prop.name, sizeof ctx->name - 1);
  *out = ctx;
  return FRW_OK;
}

void frw_ctx_destroy(frw_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  frw_nccl_destroy(ctx);
  if (ctx->walk_free) ctx->walk_free(ctx);
  auto& g = ctx->grid;
  cudaFree(g.d_map);  // also releases d_rec (same allocation)
  cudaFree(g.d_full);
  cudaFree(g.d_exit);
  cudaFree(g.d_dc);
  cudaFree(g.d_mask);
  cudaFree(ctx->d_ctr);
  cudaFree(ctx->d_err);
  cudaFree(ctx->d_hist);
  cudaFree(ctx->d_mom);
  cudaFree(ctx->d_tr);
  cudaFree(ctx->d_solve);
  cudaEventDestroy(ctx->ev[0]);
  cudaEventDestroy(ctx->ev[1]);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* frw_last_error(const frw_ctx* ctx) {
  return ctx ? ctx->err.c_str() : "null context";
}

int frw_device_info(const frw_ctx* ctx, int* sm_count, int* sm_clock_khz,
                    char* name, int name_len) {
  if (!ctx) return FRW_EINVAL;
  if (sm_count) *sm_count = ctx->sm_count;
  if (sm_clock_khz) *sm_clock_khz = ctx->sm_clock_khz;
  if (name && name_len > 0) {
    std::strncpy(name, ctx->name, name_len - 1);
    name[name_len - 1] = 0;
  }
  return FRW_OK;
}

int frw_set_stream(frw_ctx* ctx, void* stream) {
  if (!ctx) return FRW_EINVAL;
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  ctx->stream = static_cast<cudaStream_t>(stream);
  ctx->own_stream = false;
  return FRW_OK;
}

int frw_synchronize(frw_ctx* ctx) {
  if (!ctx) return FRW_EINVAL;
  FRW_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return FRW_OK;
}

int frw_event_record(frw_ctx* ctx, int which) {
  if (!ctx || which < 0 || which > 1) return FRW_EINVAL;
  FRW_CUDA(ctx, cudaEventRecord(ctx->ev[which], ctx->stream));
  return FRW_OK;
}

int frw_event_elapsed_ms(frw_ctx* ctx, float* ms) {
  if (!ctx || !ms) return FRW_EINVAL;
  FRW_CUDA(ctx, cudaEventSynchronize(ctx->ev[1]));
  FRW_CUDA(ctx, cudaEventElapsedTime(ms, ctx->ev[0], ctx->ev[1]));
  return FRW_OK;
}

int frw_dev_alloc(frw_ctx* ctx, size_t bytes, void** ptr) {
  if (!ctx || !ptr) return FRW_EINVAL;
  FRW_CUDA(ctx, cudaSetDevice(ctx->device));
  FRW_CUDA(ctx, cudaMalloc(ptr, bytes));
  return FRW_OK;
}

int frw_dev_free(frw_ctx* ctx, void* ptr) {
  if (!ctx) return FRW_EINVAL;
  FRW_CUDA(ctx, cudaFree(ptr));
  return FRW_OK;
}

int frw_host_alloc(frw_ctx* ctx, size_t bytes, void** ptr) {
  if (!ctx || !ptr) return FRW_EINVAL;
  FRW_CUDA(ctx, cudaSetDevice(ctx->device));
  FRW_CUDA(ctx, cudaMallocHost(ptr, bytes));
  return FRW_OK;
}

int frw_host_free(frw_ctx* ctx, void* ptr) {
  if (!ctx) return FRW_EINVAL;
  FRW_CUDA(ctx, cudaFreeHost(ptr));
  return FRW_OK;
}

int frw_dev_memset(frw_ctx* ctx, void* ptr, int value, size_t bytes) {
  if (!ctx) return FRW_EINVAL;
  FRW_CUDA(ctx, cudaMemsetAsync(ptr, value, bytes, ctx->stream));
  return FRW_OK;
}

int frw_memcpy_h2d(frw_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (!ctx) return FRW_EINVAL;
  FRW_CUDA(ctx, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  FRW_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return FRW_OK;
}

int frw_memcpy_d2h(frw_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (!ctx) return FRW_EINVAL;
  FRW_CUDA(ctx, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  FRW_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return FRW_OK;
}

int frw_smem_bandwidth_probe(frw_ctx* ctx, int iters, double* bytes_per_s) {
  if (!ctx || !bytes_per_s || iters < 1) return FRW_EINVAL;
  uint32_t* sink = nullptr;
  FRW_CUDA(ctx, cudaMalloc(&sink, 16));
  const int blocks = ctx->sm_count * 2;
  smem_probe_kernel<<<blocks, 1024, 0, ctx->stream>>>(iters, sink);  // warm
  FRW_CUDA(ctx, cudaEventRecord(ctx->ev[0], ctx->stream));
  smem_probe_kernel<<<blocks, 1024, 0, ctx->stream>>>(iters, sink);
  FRW_CUDA(ctx, cudaEventRecord(ctx->ev[1], ctx->stream));
  FRW_CUDA(ctx, cudaEventSynchronize(ctx->ev[1]));
  float ms = 0;
  FRW_CUDA(ctx, cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]));
  cudaFree(sink);
  *bytes_per_s = double(blocks) * 1024.0 * iters * 8 * 16 / (ms * 1e-3);
  return FRW_OK;
}

}  // extern "C"
