// Per-instruction issue cost on B200 (tuning probe): 8 independent chains per
// thread of one integer op, 64 warps per SM; prints warp-instructions per
// cycle per SM sub-partition (1.0 = one per clock, 0.5 = a 2-cycle pipe).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int OP>
__global__ void __launch_bounds__(1024, 2) k(uint32_t* out, uint32_t s, int iters) {
  uint32_t a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * (j + 3) + s;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t x = a[j];
      if (OP == 0) asm volatile("mad.lo.u32 %0, %0, 0x1ce4e5b9, %1;" : "+r"(x) : "r"(s));
      if (OP == 1) { uint64_t w; asm volatile("mul.wide.u32 %0, %1, 0x1ce4e5b9;" : "=l"(w) : "r"(x)); x = (uint32_t)w ^ (uint32_t)(w >> 32); }
      if (OP == 2) asm volatile("mad.hi.u32 %0, %0, 0x1ce4e5b9, %1;" : "+r"(x) : "r"(s));
      if (OP == 3) asm volatile("shf.r.wrap.b32 %0, %0, %1, 27;" : "+r"(x) : "r"(s));
      if (OP == 4) asm volatile("lop3.b32 %0, %0, %1, 0x1234, 0x96;" : "+r"(x) : "r"(s));
      if (OP == 5) asm volatile("add.u32 %0, %0, %1;" : "+r"(x) : "r"(s));
      if (OP == 6) asm volatile("shr.u32 %0, %0, 27;" : "+r"(x));
      a[j] = x;
    }
  }
  uint32_t r = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) r ^= a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
int main() {
  int sms = 148, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t* out;
  cudaMalloc(&out, 4ull * 2 * sms * 1024);
  const int iters = 4096;
  const char* names[7] = {"IMAD", "IMAD.WIDE(+LOP3)", "IMAD.HI", "SHF.R.W", "LOP3", "IADD", "SHR"};
  for (int op = 0; op < 7; ++op) {
    auto launch = [&]() {
      switch (op) {
        case 0: k<0><<<2 * sms, 1024>>>(out, 7, iters); break;
        case 1: k<1><<<2 * sms, 1024>>>(out, 7, iters); break;
        case 2: k<2><<<2 * sms, 1024>>>(out, 7, iters); break;
        case 3: k<3><<<2 * sms, 1024>>>(out, 7, iters); break;
        case 4: k<4><<<2 * sms, 1024>>>(out, 7, iters); break;
        case 5: k<5><<<2 * sms, 1024>>>(out, 7, iters); break;
        case 6: k<6><<<2 * sms, 1024>>>(out, 7, iters); break;
      }
    };
    launch();
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double winst = (double)2 * sms * 32 * iters * 8;  // warp-instructions of the op (per SM: /sms)
    const double cycles = ms * 1e-3 * 1965e6;                  // B200 boost clock
    printf("{\"op\": \"%s\", \"warp_inst_per_cycle_per_smsp\": %.3f, \"ms\": %.3f}\n", names[op],
           winst / sms / 4 / cycles, ms);
  }
  return 0;
}
