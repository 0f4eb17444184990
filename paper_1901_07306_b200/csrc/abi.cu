// Library identity, host-side helpers and the roofline microbenchmark.
#include <cstring>
#include <cuda_runtime.h>
#include "sspd_common.cuh"
#include "launch.cuh"

namespace sspd {

__device__ __forceinline__ uint32_t xorshift(uint32_t& s) {
  s ^= s << 13;
  s ^= s >> 17;
  s ^= s << 5;
  return s;
}

// Random red.global.or.b32 over a power-of-two word buffer: the L2-atomic
// term of the scan roofline, issued with the scan's
// instruction (red.relaxed.gpu.global.or.b32).
__global__ void __launch_bounds__(256) microbench_red_kernel(uint32_t* buf, uint32_t words_mask, int iters) {
  uint32_t s = 0x9E3779B9u ^ ((blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u);
  for (int i = 0; i < iters; ++i) {
    const uint32_t r = xorshift(s);
    asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(buf + (r & words_mask)), "r"(1u << (r >> 27))
                 : "memory");
  }
}

// Random u16 stores with the sliding scan's instruction (st.global.u16) over
// a `bytes` footprint: the roofline term of K2 (the pool is
// not L2-resident, so every stamp store is a partial-sector write).
__global__ void __launch_bounds__(256) microbench_store16_kernel(uint16_t* buf, uint32_t elems_mask, int iters) {
  uint32_t s = 0x2545F491u ^ ((blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u);
  for (int i = 0; i < iters; ++i) {
    const uint32_t r = xorshift(s);
    asm volatile("st.global.u16 [%0], %1;" ::"l"(buf + (r & elems_mask)), "h"((unsigned short)(r >> 16)) : "memory");
  }
}

}  // namespace sspd

using namespace sspd;

extern "C" int sspd_abi_version(void) { return SSPD_ABI_VERSION; }

extern "C" size_t sspd_params_size(void) { return sizeof(sspd_params); }

extern "C" int sspd_device_sm_count(int device) {
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return n;
}

extern "C" uint64_t sspd_mix64_host(uint64_t x) { return mix64(x); }

extern "C" uint64_t sspd_hash_range_host(uint64_t key, uint64_t seed, const sspd_divisor* d) {
  return hash_range(key, seed, *d);
}

extern "C" int sspd_microbench_red(void* buf, uint64_t bytes, int blocks_per_sm, int iters, double* ops_per_s,
                                   void* stream) {
  if (!buf || !ops_per_s || bytes < 4 || (bytes & (bytes - 1))) return SSPD_ERR_CONFIG;
  if (bytes / 4 - 1 > 0xFFFFFFFFull) return SSPD_ERR_CONFIG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = sms * (blocks_per_sm > 0 ? blocks_per_sm : 8);
  const uint32_t mask = (uint32_t)(bytes / 4 - 1);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  microbench_red_kernel<<<grid, 256, 0, st>>>(static_cast<uint32_t*>(buf), mask, iters);  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a, st);
    microbench_red_kernel<<<grid, 256, 0, st>>>(static_cast<uint32_t*>(buf), mask, iters);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  *ops_per_s = (double)grid * 256.0 * iters / (best * 1e-3);
  return check_launch();
}

extern "C" int sspd_microbench_store16(void* buf, uint64_t bytes, int blocks_per_sm, int iters, double* ops_per_s,
                                       void* stream) {
  if (!buf || !ops_per_s || bytes < 2 || (bytes & (bytes - 1))) return SSPD_ERR_CONFIG;
  if (bytes / 2 - 1 > 0xFFFFFFFFull) return SSPD_ERR_CONFIG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = sms * (blocks_per_sm > 0 ? blocks_per_sm : 8);
  const uint32_t mask = (uint32_t)(bytes / 2 - 1);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  microbench_store16_kernel<<<grid, 256, 0, st>>>(static_cast<uint16_t*>(buf), mask, iters);  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a, st);
    microbench_store16_kernel<<<grid, 256, 0, st>>>(static_cast<uint16_t*>(buf), mask, iters);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  *ops_per_s = (double)grid * 256.0 * iters / (best * 1e-3);
  return check_launch();
}

// ---- CUDA IPC plumbing for the multi-GPU OR-merge (multigpu.py) --------
// A rank's sketch block is one cudaMalloc allocation so that its IPC
// handle maps exactly that block into every peer process.
extern "C" int sspd_ipc_alloc(uint64_t bytes, void** ptr) {
  if (!ptr || bytes == 0) return SSPD_ERR_DATA;
  if (cudaMalloc(ptr, bytes) != cudaSuccess) return SSPD_ERR_CUDA;
  if (cudaMemset(*ptr, 0, bytes) != cudaSuccess) return SSPD_ERR_CUDA;
  return SSPD_OK;
}

extern "C" int sspd_ipc_free(void* ptr) { return cudaFree(ptr) == cudaSuccess ? SSPD_OK : SSPD_ERR_CUDA; }

extern "C" int sspd_ipc_get_handle(void* ptr, uint8_t* handle_out) {
  if (!ptr || !handle_out) return SSPD_ERR_DATA;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, ptr) != cudaSuccess) return SSPD_ERR_CUDA;
  memcpy(handle_out, &h, sizeof(h));
  return SSPD_OK;
}

extern "C" int sspd_ipc_open(const uint8_t* handle, void** ptr) {
  if (!handle || !ptr) return SSPD_ERR_DATA;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  if (cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
    cudaGetLastError();
    return SSPD_ERR_CUDA;
  }
  return SSPD_OK;
}

extern "C" int sspd_ipc_close(void* ptr) {
  return cudaIpcCloseMemHandle(ptr) == cudaSuccess ? SSPD_OK : SSPD_ERR_CUDA;
}

extern "C" int sspd_copy_async(void* dst, const void* src, uint64_t bytes, void* stream) {
  if (bytes == 0) return SSPD_OK;
  return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, static_cast<cudaStream_t>(stream)) == cudaSuccess
             ? SSPD_OK
             : SSPD_ERR_CUDA;
}
