// Exact per-host distinct-peer counts on the GPU -- the reference's
// ExactOracle (sspd/evaluation.py:32-58): sort-unique of the u64 keys
// (hip << 32 | oip), then the distinct keys counted per host.
//
// Evaluation infrastructure for the large configs,
// where the reference's np.unique over 2^28+ keys takes minutes on the
// host.  Not on the scan path.  Algorithm:
//   1. pack      keys[i] = hip_i << 32 | oip_i                (coalesced)
//   2. sort      CUB radix sort of the 64-bit keys
//   3. mark      host[i] = key[i] >> 32, fresh[i] = key[i] != key[i-1]
//   4. reduce    per run of equal host: sum(fresh)  (CUB reduce-by-key)
// giving hosts ascending (np.unique order) with their distinct counts.
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include "launch.cuh"

namespace sspd {

__global__ void pack_keys_kernel(const uint32_t* __restrict__ hips, const uint32_t* __restrict__ oips, uint64_t n,
                                 uint64_t* __restrict__ keys) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    keys[i] = ((uint64_t)__ldcs(hips + i) << 32) | __ldcs(oips + i);
}

__global__ void mark_runs_kernel(const uint64_t* __restrict__ sorted, uint64_t n, uint32_t* __restrict__ host,
                                 uint32_t* __restrict__ fresh) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = sorted[i];
    host[i] = (uint32_t)(v >> 32);
    fresh[i] = (i == 0 || sorted[i - 1] != v) ? 1u : 0u;
  }
}

struct ExactLayout {
  size_t keys_b, host, fresh, temp, temp_bytes, total;
};

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static int exact_layout(uint64_t n, cudaStream_t st, ExactLayout& L) {
  const int ni = (int)(n ? n : 1);
  size_t sort_tmp = 0, rbk_tmp = 0;
  cub::DoubleBuffer<uint64_t> kb(nullptr, nullptr);
  if (cub::DeviceRadixSort::SortKeys(nullptr, sort_tmp, kb, ni, 0, 64, st) != cudaSuccess) return SSPD_ERR_CUDA;
  if (cub::DeviceReduce::ReduceByKey(nullptr, rbk_tmp, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                     (const uint32_t*)nullptr, (uint32_t*)nullptr, (unsigned long long*)nullptr,
                                     cub::Sum(), ni, st) != cudaSuccess)
    return SSPD_ERR_CUDA;
  L.temp_bytes = sort_tmp > rbk_tmp ? sort_tmp : rbk_tmp;
  // [keys_a | keys_b | host | fresh | temp]
  L.keys_b = align256(8 * (size_t)ni);
  L.host = L.keys_b + align256(8 * (size_t)ni);
  L.fresh = L.host + align256(4 * (size_t)ni);
  L.temp = L.fresh + align256(4 * (size_t)ni);
  L.total = L.temp + align256(L.temp_bytes);
  return SSPD_OK;
}

}  // namespace sspd

using namespace sspd;

extern "C" int sspd_exact_cardinalities(const uint32_t* hips, const uint32_t* oips, uint64_t n, uint32_t* hosts_out,
                                        uint32_t* counts_out, unsigned long long* n_hosts_out, void* scratch,
                                        size_t* scratch_bytes, void* stream) {
  if (!scratch_bytes) return SSPD_ERR_DATA;
  if (n >= (1ull << 31)) return SSPD_ERR_CONFIG;  // CUB item counts are int
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ExactLayout L;
  if (int rc = exact_layout(n, st, L)) return rc;
  if (!scratch) {
    *scratch_bytes = L.total;
    return SSPD_OK;
  }
  if (*scratch_bytes < L.total) return SSPD_ERR_CAPACITY;
  if (!n_hosts_out) return SSPD_ERR_DATA;
  if (n == 0) return cudaMemsetAsync(n_hosts_out, 0, sizeof(unsigned long long), st) == cudaSuccess ? SSPD_OK
                                                                                                    : SSPD_ERR_CUDA;
  if (!hips || !oips || !hosts_out || !counts_out) return SSPD_ERR_DATA;
  uint8_t* s = static_cast<uint8_t*>(scratch);
  uint64_t* keys_a = reinterpret_cast<uint64_t*>(s);
  uint64_t* keys_b = reinterpret_cast<uint64_t*>(s + L.keys_b);
  uint32_t* host = reinterpret_cast<uint32_t*>(s + L.host);
  uint32_t* fresh = reinterpret_cast<uint32_t*>(s + L.fresh);
  void* temp = s + L.temp;
  size_t temp_bytes = L.temp_bytes;
  pack_keys_kernel<<<grid_for(pack_keys_kernel, 256, n), 256, 0, st>>>(hips, oips, n, keys_a);
  cub::DoubleBuffer<uint64_t> kb(keys_a, keys_b);
  if (cub::DeviceRadixSort::SortKeys(temp, temp_bytes, kb, (int)n, 0, 64, st) != cudaSuccess) return SSPD_ERR_CUDA;
  mark_runs_kernel<<<grid_for(mark_runs_kernel, 256, n), 256, 0, st>>>(kb.Current(), n, host, fresh);
  temp_bytes = L.temp_bytes;
  if (cub::DeviceReduce::ReduceByKey(temp, temp_bytes, host, hosts_out, fresh, counts_out, n_hosts_out, cub::Sum(),
                                     (int)n, st) != cudaSuccess)
    return SSPD_ERR_CUDA;
  return check_launch();
}
