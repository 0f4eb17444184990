// Grid-barrier latency on one B200: cooperative-groups grid.sync() vs a
// sense-reversing barrier polled with ld.acquire.gpu, 148 x 1024 threads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gridsync_bench gridsync_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, unsigned* sink) {
  cg::grid_group g = cg::this_grid();
  unsigned acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += threadIdx.x ^ i;
    g.sync();
  }
  if (acc == 0xFFFFFFFFu) *sink = acc;
}

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__global__ void k_custom(int iters, unsigned* count, unsigned* gen, unsigned* sink) {
  unsigned acc = 0;
  const unsigned nb = gridDim.x;
  for (int i = 0; i < iters; ++i) {
    acc += threadIdx.x ^ i;
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned g = ld_acq(gen);
      if (atom_add_acqrel(count, 1u) == nb - 1) {
        *count = 0;
        st_rel(gen, g + 1);
      } else {
        while (ld_acq(gen) == g) {
        }
      }
    }
    __syncthreads();
  }
  if (acc == 0xFFFFFFFFu) *sink = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *buf;
  cudaMalloc(&buf, 64);
  cudaMemset(buf, 0, 64);
  const int iters = 2000;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    int it = iters;
    unsigned* sink = buf + 8;
    void* args[] = {&it, &sink};
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_cg, dim3(sms), dim3(1024), args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"barrier\": \"cg::grid.sync\", \"us_per_sync\": %.3f}\n", ms * 1000 / iters);
    unsigned *cnt = buf, *gen = buf + 4;
    void* args2[] = {&it, &cnt, &gen, &sink};
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_custom, dim3(sms), dim3(1024), args2, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"barrier\": \"custom acq/rel\", \"us_per_sync\": %.3f}\n", ms * 1000 / iters);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
