// Round-1 design probe #2: can the scan beat the L2 RED rate?
//  (a) random loads (ld.global / ld.global.nc) from an L2-resident buffer,
//  (b) check-before-set: load the word, issue red.or only if the bit is clear,
//      at several "already set" fractions,
//  (c) a scan-shaped kernel with 8 row updates per packet done as
//      load-check-red.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t xs(uint32_t& s) { s ^= s << 13; s ^= s >> 17; s ^= s << 5; return s; }

template <int kNc>
__global__ void k_ld(const uint32_t* buf, uint32_t mask, int iters, uint32_t* out) {
  uint32_t s = 0x9E3779B9u ^ (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
  uint32_t acc = 0;
  for (int i = 0; i < iters; i += 8) {
    uint32_t v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t r = xs(s);
      const uint32_t* p = buf + (r & mask);
      if (kNc) asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v[j]) : "l"(p));
      else asm volatile("ld.global.relaxed.gpu.u32 %0, [%1];" : "=r"(v[j]) : "l"(p));
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += v[j];
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// buffer pre-filled so a fraction of bits is set; check-before-set
template <int kNc>
__global__ void k_check_red(uint32_t* buf, uint32_t mask, int iters) {
  uint32_t s = 0x1234567u ^ (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
  for (int i = 0; i < iters; i += 8) {
    uint32_t addr[8], bit[8], v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t r = xs(s);
      addr[j] = r & mask;
      bit[j] = 1u << (xs(s) & 31);
      const uint32_t* p = buf + addr[j];
      if (kNc) asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v[j]) : "l"(p));
      else asm volatile("ld.global.relaxed.gpu.u32 %0, [%1];" : "=r"(v[j]) : "l"(p));
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (!(v[j] & bit[j]))
        asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(buf + addr[j]), "r"(bit[j]) : "memory");
  }
}

__global__ void k_plain_red(uint32_t* buf, uint32_t mask, int iters) {
  uint32_t s = 0x1234567u ^ (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
  for (int i = 0; i < iters; ++i) {
    uint32_t r = xs(s);
    uint32_t b = 1u << (xs(s) & 31);
    asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(buf + (r & mask)), "r"(b) : "memory");
  }
}

__global__ void k_fill(uint32_t* buf, uint32_t n, uint32_t thresh) {  // each bit set with P = thresh/2^32
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t s = 0xABCDu ^ (i * 2654435761u) ^ 0x55555555u;
  uint32_t w = 0;
  for (int b = 0; b < 32; ++b) if (xs(s) < thresh) w |= 1u << b;
  buf[i] = w;
}

int main() {
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint32_t* buf; CK(cudaMalloc(&buf, 64u << 20));
  uint32_t* out; CK(cudaMalloc(&out, 4096));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto timeit = [&](const char* name, double ops, auto launch, auto prep) {
    prep(); launch(); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      prep();
      cudaEventRecord(a); launch(); cudaEventRecord(b); CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    CK(cudaGetLastError());
    printf("{\"bench\": \"%s\", \"ms\": %.4f, \"Gops\": %.2f}\n", name, best, ops / best / 1e6);
    fflush(stdout);
  };
  const int T = 256, grid = sms * 8;
  auto noprep = [] {};
  for (uint32_t mb : {8u, 64u}) {
    uint32_t words = (mb << 20) / 4;
    char nm[128];
    snprintf(nm, 128, "ld.relaxed random %uMiB", mb);
    timeit(nm, (double)grid * T * 512, [&] { k_ld<0><<<grid, T>>>(buf, words - 1, 512, out); }, noprep);
    snprintf(nm, 128, "ld.nc random %uMiB", mb);
    timeit(nm, (double)grid * T * 512, [&] { k_ld<1><<<grid, T>>>(buf, words - 1, 512, out); }, noprep);
    for (double frac : {0.0, 0.5, 0.9, 0.99}) {
      uint32_t thresh = (uint32_t)(frac * 4294967295.0);
      auto prep = [&] { k_fill<<<(words + 255) / 256, 256>>>(buf, words, thresh); };
      snprintf(nm, 128, "plain red %uMiB preset=%.2f", mb, frac);
      timeit(nm, (double)grid * T * 256, [&] { k_plain_red<<<grid, T>>>(buf, words - 1, 256); }, prep);
      snprintf(nm, 128, "check(ld)+red %uMiB preset=%.2f", mb, frac);
      timeit(nm, (double)grid * T * 256, [&] { k_check_red<0><<<grid, T>>>(buf, words - 1, 256); }, prep);
      snprintf(nm, 128, "check(ld.nc)+red %uMiB preset=%.2f", mb, frac);
      timeit(nm, (double)grid * T * 256, [&] { k_check_red<1><<<grid, T>>>(buf, words - 1, 256); }, prep);
    }
  }
  return 0;
}
