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

// The scan's compute floor: stream (hip, oip) pairs with the scan's 16-byte
// loads and evaluate exactly the hashes the partitioned scans evaluate per
// packet -- H3 % k, the H1 sampling test and LR row hashes % lc (split-seed
// SplitMix64, sspd_common.cuh) -- with no sketch update at all.  The packets/s
// it reaches bound any scan that must compute these indexes (SURVEY.md
// §8(a) a1-a2): K1b is issue-bound on exactly this work.
struct HashSeeds {
  SplitSeed ss[2 + SSPD_MAX_LR];
  uint32_t lr, k_mask, lc_mask, tmask;
};

template <int kMinBlocks, int kLRc>
__global__ void __launch_bounds__(1024, kMinBlocks)
    microbench_hash_kernel(const uint32_t* __restrict__ hips, const uint32_t* __restrict__ oips, uint64_t nq,
                           const __grid_constant__ HashSeeds S, uint32_t* sink) {
  uint32_t acc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += stride) {
    const uint4 hv = __ldcs(reinterpret_cast<const uint4*>(hips) + q);
    const uint4 ov = __ldcs(reinterpret_cast<const uint4*>(oips) + q);
    const uint32_t h[4] = {hv.x, hv.y, hv.z, hv.w}, o[4] = {ov.x, ov.y, ov.z, ov.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint32_t v = mix64_lo_fast(o[e], S.ss[0]) & S.k_mask;
      v ^= (mix64_lo_fast(o[e], S.ss[1]) & S.tmask) == 0u ? 0x80000000u : 0u;
      const uint32_t lr = kLRc ? kLRc : S.lr;  // LR = 8 (the scans' compile-time rows): seeds as constant operands
#pragma unroll 8
      for (uint32_t i = 0; i < lr; ++i) v += (mix64_lo_fast(h[e], S.ss[2 + i]) & S.lc_mask) << i;
      acc ^= v;
    }
  }
  sink[(uint64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

}  // namespace sspd

using namespace sspd;

// Hash-floor packets/s of the scans over the caller's packets (n % 4 == 0
// used, 16-byte aligned), at `blocks_per_sm` CTAs of 1,024 threads per SM
// (1 = the partitioned scans' launch shape, 2 = full occupancy: 32
// registers per thread); sink: >= 2048 * SMs words.  Best of 5 after one
// warm-up.
extern "C" int sspd_microbench_hash(const uint32_t* hips, const uint32_t* oips, uint64_t n, const sspd_params* p,
                                    int blocks_per_sm, uint32_t* sink, double* pkts_per_s, void* stream) {
  int rc = validate_params(p);
  if (rc) return rc;
  if (!hips || !oips || !sink || !pkts_per_s || n < 4) return SSPD_ERR_DATA;
  if (((reinterpret_cast<uintptr_t>(hips) | reinterpret_cast<uintptr_t>(oips)) & 15u) != 0) return SSPD_ERR_DATA;
  if ((p->k & (p->k - 1)) || (p->lc & (p->lc - 1))) return SSPD_ERR_CONFIG;  // masks, as the scans' fast modes
  if (blocks_per_sm != 1 && blocks_per_sm != 2) return SSPD_ERR_CONFIG;
  HashSeeds S;
  const uint64_t seeds[2] = {p->seed_h3, p->seed_h1};
  for (int i = 0; i < 2 + (int)p->lr; ++i) {
    const uint64_t sd = i < 2 ? seeds[i] : p->seed_lh[i - 2];
    S.ss[i] = split_seed(sd);
  }
  S.lr = p->lr;
  S.k_mask = p->k - 1;
  S.lc_mask = p->lc - 1;
  S.tmask = tau_mask(p->tau);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t nq = n / 4;
  const int threads = 1024, grid = sms * blocks_per_sm;
  auto launch = [&]() {
    const bool lr8 = S.lr == 8;
    if (blocks_per_sm == 1 && lr8)
      microbench_hash_kernel<1, 8><<<grid, threads, 0, st>>>(hips, oips, nq, S, sink);
    else if (blocks_per_sm == 1)
      microbench_hash_kernel<1, 0><<<grid, threads, 0, st>>>(hips, oips, nq, S, sink);
    else if (lr8)
      microbench_hash_kernel<2, 8><<<grid, threads, 0, st>>>(hips, oips, nq, S, sink);
    else
      microbench_hash_kernel<2, 0><<<grid, threads, 0, st>>>(hips, oips, nq, S, sink);
  };
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a, st);
    launch();
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  *pkts_per_s = (double)(nq * 4) / (best * 1e-3);
  return check_launch();
}

// ---- the scans' 32-bit hash against the 64-bit definition --------------
// Every 32-bit key k in [key0, key0 + nkeys): mix64_lo_fast(k, split_seed(seed))
// == (uint32_t)mix64(k ^ seed) (hashing.py:48-53).  Mismatches are counted
// and the smallest mismatching key is kept (0xFFFFFFFFFFFFFFFF when none).
__global__ void check_mix_kernel(uint64_t seed, SplitSeed ss, uint64_t key0, uint64_t nkeys,
                                 unsigned long long* out) {
  uint32_t bad = 0;
  unsigned long long first = ~0ull;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nkeys; i += stride) {
    const uint32_t k = (uint32_t)(key0 + i);
    if (mix64_lo_fast(k, ss) != (uint32_t)mix64((uint64_t)k ^ seed)) {
      ++bad;
      first = min(first, (unsigned long long)k);
    }
  }
  if (bad) {
    atomicAdd(out, (unsigned long long)bad);
    atomicMin(out + 1, first);
  }
}

extern "C" int sspd_check_hash32(uint64_t seed, uint64_t key0, uint64_t nkeys, uint64_t* mismatches,
                                 uint64_t* first_bad, void* stream) {
  if (!mismatches || !first_bad || key0 + nkeys > (1ull << 32) || nkeys == 0) return SSPD_ERR_DATA;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, 16) != cudaSuccess) return SSPD_ERR_CUDA;
  const unsigned long long init[2] = {0ull, ~0ull};
  cudaMemcpyAsync(d, init, 16, cudaMemcpyHostToDevice, st);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  check_mix_kernel<<<sms * 8, 256, 0, st>>>(seed, split_seed(seed), key0, nkeys, d);
  unsigned long long h[2];
  cudaMemcpyAsync(h, d, 16, cudaMemcpyDeviceToHost, st);
  const cudaError_t e = cudaStreamSynchronize(st);
  cudaFree(d);
  if (e != cudaSuccess) return SSPD_ERR_CUDA;
  *mismatches = h[0];
  *first_bad = h[1];
  return check_launch();
}

// ---- host staging of caller arrays (DetectorState.process_batch from host
// memory): IPv4 keys of any integer width narrowed to u32 in one pass, so a
// 65,536-pair numpy batch costs one read + one write of host memory.
template <typename T>
static int check_u32_range(const T* s, uint64_t n) {
  uint64_t bad = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t v = (uint64_t)s[i];  // negative values wrap to >= 2^63
    bad |= v >> 32;
  }
  return bad ? SSPD_ERR_DATA : SSPD_OK;
}

extern "C" int sspd_host_check_u32(const void* src, uint64_t n, uint32_t elem_bytes, int is_signed) {
  if (n == 0) return SSPD_OK;
  if (!src) return SSPD_ERR_DATA;
  switch (elem_bytes * 2 + (is_signed ? 1 : 0)) {
    case 2: case 4: return SSPD_OK;                              // u8 / u16
    case 3: return check_u32_range(static_cast<const int8_t*>(src), n);
    case 5: return check_u32_range(static_cast<const int16_t*>(src), n);
    case 8: return SSPD_OK;                                      // u32
    case 9: return check_u32_range(static_cast<const int32_t*>(src), n);
    case 16: return check_u32_range(static_cast<const uint64_t*>(src), n);
    case 17: return check_u32_range(static_cast<const int64_t*>(src), n);
    default: return SSPD_ERR_CONFIG;
  }
}

template <typename T>
static void pack_u32(const T* s, uint64_t n, uint32_t* d) {
  for (uint64_t i = 0; i < n; ++i) d[i] = (uint32_t)s[i];
}

extern "C" int sspd_host_pack_u32(const void* src, uint64_t n, uint32_t elem_bytes, int is_signed, uint32_t* dst) {
  if (n == 0) return SSPD_OK;
  if (!src || !dst) return SSPD_ERR_DATA;
  switch (elem_bytes) {
    case 1: pack_u32(static_cast<const uint8_t*>(src), n, dst); break;
    case 2: pack_u32(static_cast<const uint16_t*>(src), n, dst); break;
    case 4: memcpy(dst, src, n * 4); break;
    case 8: pack_u32(static_cast<const uint64_t*>(src), n, dst); break;
    default: return SSPD_ERR_CONFIG;
  }
  (void)is_signed;  // the bit pattern of a checked key is the same either way
  return SSPD_OK;
}

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
