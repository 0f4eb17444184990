// Standalone B200 microbenchmarks that size the packet-scan roofline:
// random-address L2 RED/atomics, plain byte stores, shared-memory atomics,
// DSMEM reds, and the integer cost of the SplitMix64 hash.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o l2_microbench l2_microbench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t xs(uint32_t& s) { s ^= s << 13; s ^= s >> 17; s ^= s << 5; return s; }

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// 1) random red.global.or.b32 over a (pow2) word buffer
__global__ void k_red_or(uint32_t* buf, uint32_t mask_words, int iters) {
  uint32_t s = 0x9E3779B9u ^ (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
  for (int i = 0; i < iters; ++i) {
    uint32_t r = xs(s);
    asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" :: "l"(buf + (r & mask_words)), "r"(1u << (r >> 27)) : "memory");
  }
}
// 1b) 8 reds per "packet" sharing one bit, rows of 1/8 of buffer (scan-shaped)
__global__ void k_red_or_rows(uint32_t* buf, uint32_t row_words_mask, uint32_t row_words, int iters) {
  uint32_t s = 0x1234567u ^ (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
  for (int i = 0; i < iters; ++i) {
    uint32_t b = xs(s);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      uint32_t c = xs(s);
      asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" :: "l"(buf + r * row_words + (c & row_words_mask)), "r"(1u << (b & 31)) : "memory");
    }
  }
}
// 2) random plain byte store over a byte buffer (byte-per-bit layout)
__global__ void k_st_u8(uint8_t* buf, uint32_t mask_bytes, int iters) {
  uint32_t s = 0x9E3779B9u ^ (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
  for (int i = 0; i < iters; ++i) {
    uint32_t r = xs(s);
    asm volatile("st.global.u8 [%0], %1;" :: "l"(buf + (r & mask_bytes)), "h"((unsigned short)1) : "memory");
  }
}
// 2b) random u16 store (sliding timestamps)
__global__ void k_st_u16(uint16_t* buf, uint32_t mask_elems, int iters) {
  uint32_t s = 0x9E3779B9u ^ (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
  for (int i = 0; i < iters; ++i) {
    uint32_t r = xs(s);
    asm volatile("st.global.u16 [%0], %1;" :: "l"(buf + (r & mask_elems)), "h"((unsigned short)7) : "memory");
  }
}
// 3) random shared-memory atomicOr in a per-CTA table
__global__ void k_smem_or(uint32_t* out, uint32_t words_mask, int iters) {
  extern __shared__ uint32_t sm[];
  for (uint32_t i = threadIdx.x; i <= words_mask; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  uint32_t s = 0x9E3779B9u ^ (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
  for (int i = 0; i < iters; ++i) {
    uint32_t r = xs(s);
    atomicOr(&sm[r & words_mask], 1u << (r >> 27));
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = sm[0];
}
// 4) random shared-memory byte store
__global__ void k_smem_st8(uint32_t* out, uint32_t bytes_mask, int iters) {
  extern __shared__ uint8_t smb[];
  for (uint32_t i = threadIdx.x; i <= bytes_mask; i += blockDim.x) smb[i] = 0;
  __syncthreads();
  uint32_t s = 0x9E3779B9u ^ (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
  for (int i = 0; i < iters; ++i) {
    uint32_t r = xs(s);
    volatile uint8_t* p = smb + (r & bytes_mask);
    *p = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = smb[0];
}
// 5) DSMEM red.or to a random CTA of the cluster
__global__ void k_dsmem_or(uint32_t* out, uint32_t words_mask, int iters) {
  extern __shared__ uint32_t sm[];
  cg::cluster_group cl = cg::this_cluster();
  for (uint32_t i = threadIdx.x; i <= words_mask; i += blockDim.x) sm[i] = 0;
  cl.sync();
  uint32_t csz = cl.num_blocks();
  uint32_t base_sm = (uint32_t)__cvta_generic_to_shared(sm);
  uint32_t s = 0x9E3779B9u ^ (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
  for (int i = 0; i < iters; ++i) {
    uint32_t r = xs(s);
    uint32_t tgt = (r >> 24) % csz;
    uint32_t local = base_sm + 4u * (r & words_mask);
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(tgt));
    asm volatile("red.shared::cluster.or.b32 [%0], %1;" :: "r"(remote), "r"(1u << (r & 31)) : "memory");
  }
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = sm[0];
}
// 6) hash cost: 10 mix64 per "packet", results folded to prevent DCE
__global__ void k_hash(uint64_t* out, int iters) {
  uint64_t acc = 0;
  uint64_t x = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    uint64_t k = x + (uint64_t)i * 0x10001ull;
#pragma unroll
    for (int j = 0; j < 10; ++j) acc ^= mix64(k ^ (0x1111111111111111ull * (j + 1)));
  }
  if (acc == 0x12345) out[0] = acc;
}

int main(int argc, char** argv) {
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int l2 = 0; CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0));
  int clk = 0; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  printf("{\"sms\": %d, \"l2_bytes\": %d, \"clock_khz\": %d}\n", sms, l2, clk);
  uint8_t* big; CK(cudaMalloc(&big, 256ull << 20));
  CK(cudaMemset(big, 0, 256ull << 20));
  uint32_t* out; CK(cudaMalloc(&out, 1 << 20));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto timeit = [&](const char* name, double ops, auto launch) {
    launch(); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(a); launch(); cudaEventRecord(b); CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    CK(cudaGetLastError());
    printf("{\"bench\": \"%s\", \"ms\": %.4f, \"Gops\": %.2f}\n", name, best, ops / best / 1e6);
    fflush(stdout);
  };
  const int T = 256;
  for (int bps : {4, 8, 16}) {
    int grid = sms * bps;
    for (uint64_t mb : {8ull, 64ull}) {
      int iters = 256;
      uint32_t words = (uint32_t)(mb << 20) / 4;
      char name[96]; snprintf(name, 96, "red_or_b32 %lluMiB grid=%d", (unsigned long long)mb, grid);
      timeit(name, (double)grid * T * iters, [&] { k_red_or<<<grid, T>>>((uint32_t*)big, words - 1, iters); });
    }
  }
  {
    int grid = sms * 8, iters = 64;
    uint32_t row_words = (8u << 20) / 4 / 8;
    timeit("red_or_rows8 8MiB grid=sms*8 (ops)", (double)grid * T * iters * 8,
           [&] { k_red_or_rows<<<grid, T>>>((uint32_t*)big, row_words - 1, row_words, iters); });
    row_words = (64u << 20) / 4 / 8;
    timeit("red_or_rows8 64MiB grid=sms*8 (ops)", (double)grid * T * iters * 8,
           [&] { k_red_or_rows<<<grid, T>>>((uint32_t*)big, row_words - 1, row_words, iters); });
  }
  for (uint64_t mb : {8ull, 64ull, 128ull}) {
    int grid = sms * 8, iters = 256;
    char name[96]; snprintf(name, 96, "st_u8 %lluMiB", (unsigned long long)mb);
    timeit(name, (double)grid * T * iters, [&] { k_st_u8<<<grid, T>>>(big, (uint32_t)(mb << 20) - 1, iters); });
  }
  for (uint64_t mb : {64ull, 256ull}) {
    int grid = sms * 8, iters = 256;
    char name[96]; snprintf(name, 96, "st_u16 %lluMiB", (unsigned long long)mb);
    timeit(name, (double)grid * T * iters, [&] { k_st_u16<<<grid, T>>>((uint16_t*)big, (uint32_t)(mb << 20) / 2 - 1, iters); });
  }
  {
    int smem = 128 << 10;
    CK(cudaFuncSetAttribute(k_smem_or, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(k_smem_st8, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int grid = sms, iters = 4096;
    for (int t : {256, 512, 1024}) {
      char name[96]; snprintf(name, 96, "smem_atomicOr 128KiB/CTA T=%d", t);
      timeit(name, (double)grid * t * iters, [&] { k_smem_or<<<grid, t, smem>>>(out, smem / 4 - 1, iters); });
      snprintf(name, 96, "smem_st_u8 128KiB/CTA T=%d", t);
      timeit(name, (double)grid * t * iters, [&] { k_smem_st8<<<grid, t, smem>>>(out, smem - 1, iters); });
    }
  }
  {
    int smem = 128 << 10;
    CK(cudaFuncSetAttribute(k_dsmem_or, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(k_dsmem_or, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    for (int csz : {2, 4, 8}) {
      int grid = (sms / csz) * csz, iters = 2048, t = 1024;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid); cfg.blockDim = dim3(t); cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = csz; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      char name[96]; snprintf(name, 96, "dsmem_red_or cluster=%d", csz);
      timeit(name, (double)grid * t * iters, [&] { CK(cudaLaunchKernelEx(&cfg, k_dsmem_or, out, (uint32_t)(smem / 4 - 1), iters)); });
    }
  }
  {
    int grid = sms * 8, iters = 256;
    timeit("hash 10x mix64 (packets)", (double)grid * T * iters, [&] { k_hash<<<grid, T>>>((uint64_t*)out, iters); });
  }
  return 0;
}
