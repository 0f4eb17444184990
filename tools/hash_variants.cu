// Throughput of SplitMix64-low-word formulations on B200 (tuning probe).
// Each variant evaluates the scans' per-packet hash set (H3, H1, 8 row
// hashes) over a streamed (hip, oip) array and XORs the results into a sink;
// all variants must produce the same sink (checked).  Prints Gpps per variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hash_variants tools/hash_variants.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_1901_07306_b200/csrc/sspd_common.cuh"
using namespace sspd;

struct Seeds { SplitSeed ss[10]; };

__device__ __forceinline__ uint32_t v_old(uint32_t k, const SplitSeed& s) { return mix64_lo_split(k, s.lo, s.hg); }

// 32-bit halves, shifts on the ALU pipe, T = H0*d + e
__device__ __forceinline__ uint32_t v_shf(uint32_t key, const SplitSeed& s) {
  uint32_t l0, h0;
  asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, 0;" : "=r"(l0), "=r"(h0)
      : "r"(key ^ s.lo), "n"((uint32_t)(kGolden & 0xFFFFFFFFull)), "r"(s.hg));
  const uint32_t yl = l0 ^ __funnelshift_r(l0, h0, 30);
  const uint32_t p = yl * (uint32_t)(kMixA >> 32) + (h0 * s.d + s.e);
  const uint64_t w = (uint64_t)yl * (uint32_t)kMixA;
  const uint32_t z1l = (uint32_t)w, z1h = (uint32_t)(w >> 32) + p;
  const uint32_t y2l = z1l ^ __funnelshift_r(z1l, z1h, 27);
  const uint32_t y2h = z1h ^ (z1h >> 27);
  const uint64_t w2 = (uint64_t)y2l * (uint32_t)kMixB;
  uint32_t z2h;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(z2h) : "r"(y2l), "n"((uint32_t)(kMixB >> 32)), "r"((uint32_t)(w2 >> 32)));
  asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(z2h) : "r"(y2h), "n"((uint32_t)kMixB));
  const uint32_t z2l = (uint32_t)w2;
  return z2l ^ __funnelshift_r(z2l, z2h, 31);
}
// the same, with T and the funnel's high part picked by the carry (SEL on the ALU)
__device__ __forceinline__ uint32_t v_sel(uint32_t key, const SplitSeed& s, uint32_t t0, uint32_t t1, uint32_t f0, uint32_t f1) {
  uint32_t l0, c;
  asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, 0, 0;" : "=r"(l0), "=r"(c)
      : "r"(key ^ s.lo), "n"((uint32_t)(kGolden & 0xFFFFFFFFull)));
  const uint32_t T = c ? t1 : t0, F = c ? f1 : f0;
  const uint32_t yl = l0 ^ (l0 >> 30) ^ F;
  const uint32_t p = yl * (uint32_t)(kMixA >> 32) + T;
  const uint64_t w = (uint64_t)yl * (uint32_t)kMixA;
  const uint32_t z1l = (uint32_t)w, z1h = (uint32_t)(w >> 32) + p;
  const uint32_t y2l = z1l ^ __funnelshift_r(z1l, z1h, 27);
  const uint32_t y2h = z1h ^ (z1h >> 27);
  const uint64_t w2 = (uint64_t)y2l * (uint32_t)kMixB;
  uint32_t z2h;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(z2h) : "r"(y2l), "n"((uint32_t)(kMixB >> 32)), "r"((uint32_t)(w2 >> 32)));
  asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(z2h) : "r"(y2h), "n"((uint32_t)kMixB));
  const uint32_t z2l = (uint32_t)w2;
  return z2l ^ __funnelshift_r(z2l, z2h, 31);
}

__host__ __device__ constexpr SplitSeed split_seed_c(uint64_t seed) {
  const uint32_t lo = (uint32_t)seed, hg = (uint32_t)(seed >> 32) + (uint32_t)(kGolden >> 32), h1 = hg + 1u;
  const uint32_t t0 = (hg ^ (hg >> 30)) * (uint32_t)kMixA, t1 = (h1 ^ (h1 >> 30)) * (uint32_t)kMixA;
  return SplitSeed{lo, hg, t1 - t0, t0 - hg * (t1 - t0)};
}
// compile-time seeds (the upper bound of removing every constant-bank load)
constexpr uint64_t kSeedsC[10] = {0x9E3779B97F4A7C15ull * 3, 0x1234567ull, 0xE8AB9E9A226DF370ull, 0xD46EE1CCFC7B25FCull,
                                  0x638C62F5C9C1EAD8ull, 0x4EC976611A9CC2F7ull, 0xA8285392D2F048D4ull,
                                  0xAF77364105F4D5A6ull, 0xDF96F642FAF5ACBFull, 0x8AFCC3A11DFFAAD5ull};
template <int I>
__device__ __forceinline__ uint32_t h_imm(uint32_t key) {
  constexpr SplitSeed s = split_seed_c(kSeedsC[I]);
  return mix64_lo_fast(key, s.lo, s.hg, s.d, s.e);
}
template <int V>
__global__ void __launch_bounds__(1024, 2) kern(const uint4* __restrict__ h4, const uint4* __restrict__ o4, uint64_t nq,
                                                const __grid_constant__ Seeds S, uint32_t* sink, uint4 tt) {
  uint32_t acc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += stride) {
    const uint4 hv = __ldcs(h4 + q), ov = __ldcs(o4 + q);
    const uint32_t h[4] = {hv.x, hv.y, hv.z, hv.w}, o[4] = {ov.x, ov.y, ov.z, ov.w};
    if (V == 4) {  // seeds as immediates
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        uint32_t v = h_imm<0>(o[e]) & 8191u;
        v ^= (h_imm<1>(o[e]) & 127u) == 0u ? 0x80000000u : 0u;
        v += (h_imm<2>(h[e]) & 1023u) << 0; v += (h_imm<3>(h[e]) & 1023u) << 1;
        v += (h_imm<4>(h[e]) & 1023u) << 2; v += (h_imm<5>(h[e]) & 1023u) << 3;
        v += (h_imm<6>(h[e]) & 1023u) << 4; v += (h_imm<7>(h[e]) & 1023u) << 5;
        v += (h_imm<8>(h[e]) & 1023u) << 6; v += (h_imm<9>(h[e]) & 1023u) << 7;
        acc ^= v;
      }
      continue;
    }
    if (V == 5) {  // rows outer, packets inner: each seed's constants loaded once per 4 packets
      uint32_t v[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) v[e] = mix64_lo_fast(o[e], S.ss[0]) & 8191u;
#pragma unroll
      for (int e = 0; e < 4; ++e) v[e] ^= (mix64_lo_fast(o[e], S.ss[1]) & 127u) == 0u ? 0x80000000u : 0u;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] += (mix64_lo_fast(h[e], S.ss[2 + i]) & 1023u) << i;
      acc ^= v[0] ^ v[1] ^ v[2] ^ v[3];
      continue;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint32_t v;
      auto H = [&](uint32_t k, int i) -> uint32_t {
        if (V == 0) return v_old(k, S.ss[i]);
        if (V == 1) return mix64_lo_fast(k, S.ss[i]);
        if (V == 2) return v_shf(k, S.ss[i]);
        return v_sel(k, S.ss[i], S.ss[i].e + S.ss[i].hg * S.ss[i].d, S.ss[i].e + (S.ss[i].hg + 1) * S.ss[i].d,
                     S.ss[i].hg << 2, (S.ss[i].hg + 1) << 2);
      };
      v = H(o[e], 0) & 8191u;
      v ^= (H(o[e], 1) & 127u) == 0u ? 0x80000000u : 0u;
#pragma unroll
      for (int i = 0; i < 8; ++i) v += (H(h[e], 2 + i) & 1023u) << i;
      acc ^= v;
    }
  }
  sink[(uint64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  const uint64_t n = 1ull << 28, nq = n / 4;
  uint32_t *h, *o, *sink;
  cudaMalloc(&h, n * 4); cudaMalloc(&o, n * 4);
  int sms = 148; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = 2 * sms;
  cudaMalloc(&sink, 4ull * grid * 1024);
  // deterministic fill
  {
    uint32_t* tmp = new uint32_t[n];
    uint64_t x = 88172645463325252ull;
    for (uint64_t i = 0; i < n; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; tmp[i] = (uint32_t)x; }
    cudaMemcpy(h, tmp, n * 4, cudaMemcpyHostToDevice);
    for (uint64_t i = 0; i < n; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; tmp[i] = (uint32_t)x; }
    cudaMemcpy(o, tmp, n * 4, cudaMemcpyHostToDevice);
    delete[] tmp;
  }
  Seeds S;
  for (int i = 0; i < 10; ++i) S.ss[i] = split_seed(kSeedsC[i]);
  uint32_t* hs = new uint32_t[grid * 1024];
  uint64_t ref = 0;
  const char* names[6] = {"old_64bit_split", "fast_mulhi", "fast_shf", "fast_sel", "fast_imm_seeds", "fast_rows_outer"};
  for (int v = 0; v < 6; ++v) {
    auto launch = [&]() {
      const uint4* H4 = reinterpret_cast<const uint4*>(h);
      const uint4* O4 = reinterpret_cast<const uint4*>(o);
      uint4 tt = make_uint4(0, 0, 0, 0);
      if (v == 0) kern<0><<<grid, 1024>>>(H4, O4, nq, S, sink, tt);
      if (v == 1) kern<1><<<grid, 1024>>>(H4, O4, nq, S, sink, tt);
      if (v == 2) kern<2><<<grid, 1024>>>(H4, O4, nq, S, sink, tt);
      if (v == 3) kern<3><<<grid, 1024>>>(H4, O4, nq, S, sink, tt);
      if (v == 4) kern<4><<<grid, 1024>>>(H4, O4, nq, S, sink, tt);
      if (v == 5) kern<5><<<grid, 1024>>>(H4, O4, nq, S, sink, tt);
    };
    launch();
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e9f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    cudaMemcpy(hs, sink, 4ull * grid * 1024, cudaMemcpyDeviceToHost);
    uint64_t sum = 0;
    for (int i = 0; i < grid * 1024; ++i) sum = sum * 31 + hs[i];
    if (v == 0) ref = sum;
    printf("{\"variant\": \"%s\", \"gpps\": %.2f, \"ms\": %.4f, \"same\": %s}\n", names[v], n / (best * 1e-3) / 1e9,
           best, sum == ref ? "true" : "false");
  }
  return 0;
}
