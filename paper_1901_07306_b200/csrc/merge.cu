// K7 merge_or / K8 merge_age_min / route_pairs.
//
// The distributed reference merges watch-point frames by a bytewise OR of
// payloads (distributed.py:167-169) and sliding pools by the per-slot
// minimum wrapped age (distributed.py:176-192).  On B200 the sources are
// device buffers -- local, or a peer GPU's sketch mapped through CUDA IPC /
// peer access -- and one kernel streams all of them with 16-byte loads and
// writes the reduced stripe once.  NCCL has no bitwise-OR reduction and
// no 16-bit unsigned type, which is why this is a kernel and not a
// collective call.
#include <cuda_runtime.h>
#include "sspd_common.cuh"
#include "launch.cuh"

namespace sspd {

constexpr int kMaxSrc = 16;
struct SrcList {
  const void* p[kMaxSrc];
};

__global__ void __launch_bounds__(256) merge_or_vec_kernel(const SrcList srcs, int n_src, uint4* dst, uint64_t nvec) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nvec; j += stride) {
    uint4 acc = reinterpret_cast<const uint4*>(srcs.p[0])[j];
    for (int s = 1; s < n_src; ++s) {
      const uint4 v = reinterpret_cast<const uint4*>(srcs.p[s])[j];
      acc.x |= v.x;
      acc.y |= v.y;
      acc.z |= v.z;
      acc.w |= v.w;
    }
    dst[j] = acc;
  }
}

__global__ void __launch_bounds__(256) merge_or_byte_kernel(const SrcList srcs, int n_src, uint8_t* dst,
                                                            uint64_t begin, uint64_t end) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = begin + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < end; j += stride) {
    uint8_t acc = 0;
    for (int s = 0; s < n_src; ++s) acc |= reinterpret_cast<const uint8_t*>(srcs.p[s])[j];
    dst[j] = acc;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) merge_age_min_kernel(const SrcList srcs, int n_src, T* dst, uint64_t n,
                                                            T now) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
    T best = (T)(now - reinterpret_cast<const T*>(srcs.p[0])[j]);
    for (int s = 1; s < n_src; ++s) {
      const T age = (T)(now - reinterpret_cast<const T*>(srcs.p[s])[j]);
      best = age < best ? age : best;
    }
    dst[j] = (T)(now - best);
  }
}

__global__ void __launch_bounds__(256) route_kernel(const uint32_t* __restrict__ hips,
                                                    const uint32_t* __restrict__ oips, uint64_t n,
                                                    uint64_t seed_route, const sspd_divisor dv, int mode,
                                                    uint64_t index_base, int64_t* lanes) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
    if (mode == 0) {
      const uint64_t key = ((uint64_t)hips[j] << 32) | (uint64_t)oips[j];
      lanes[j] = (int64_t)hash_range(key, seed_route, dv);
    } else {
      lanes[j] = (int64_t)mod(index_base + j, dv);
    }
  }
}

static int merge_or_chunk(const void* const* srcs, int n_src, void* dst, uint64_t bytes, cudaStream_t st) {
  SrcList L{};
  for (int s = 0; s < n_src; ++s) L.p[s] = srcs[s];
  uintptr_t align = reinterpret_cast<uintptr_t>(dst);
  for (int s = 0; s < n_src; ++s) align |= reinterpret_cast<uintptr_t>(srcs[s]);
  uint64_t done = 0;
  if ((align & 15u) == 0 && bytes >= 16) {
    const uint64_t nvec = bytes / 16;
    const int grid = grid_for(merge_or_vec_kernel, 256, nvec);
    merge_or_vec_kernel<<<grid, 256, 0, st>>>(L, n_src, reinterpret_cast<uint4*>(dst), nvec);
    done = nvec * 16;
  }
  if (done < bytes) {
    const int grid = grid_for(merge_or_byte_kernel, 256, bytes - done);
    merge_or_byte_kernel<<<grid, 256, 0, st>>>(L, n_src, static_cast<uint8_t*>(dst), done, bytes);
  }
  return check_launch();
}

}  // namespace sspd

using namespace sspd;

extern "C" int sspd_merge_or(const void* const* srcs, int n_src, void* dst, uint64_t bytes, void* stream) {
  if (n_src < 1 || !srcs || !dst) return SSPD_ERR_DATA;
  if (bytes == 0) return SSPD_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // Fold more than kMaxSrc sources in chunks: dst accumulates (dst | next chunk).
  int rc = merge_or_chunk(srcs, n_src < kMaxSrc ? n_src : kMaxSrc, dst, bytes, st);
  for (int s = kMaxSrc; rc == SSPD_OK && s < n_src; s += kMaxSrc - 1) {
    const void* chunk[kMaxSrc];
    chunk[0] = dst;
    int m = 1;
    for (int t = s; t < n_src && m < kMaxSrc; ++t) chunk[m++] = srcs[t];
    rc = merge_or_chunk(chunk, m, dst, bytes, st);
  }
  return rc;
}

extern "C" int sspd_merge_age_min(const void* const* srcs, int n_src, void* dst, uint64_t n_slots,
                                  uint32_t ts_bytes, uint64_t now_wrapped, void* stream) {
  if (n_src < 1 || n_src > kMaxSrc || !srcs || !dst) return SSPD_ERR_DATA;
  if (n_slots == 0) return SSPD_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SrcList L{};
  for (int s = 0; s < n_src; ++s) L.p[s] = srcs[s];
  switch (ts_bytes) {
#define SSPD_AM(T)                                                                                  \
  {                                                                                                 \
    const int grid = grid_for(merge_age_min_kernel<T>, 256, n_slots);                              \
    merge_age_min_kernel<T><<<grid, 256, 0, st>>>(L, n_src, (T*)dst, n_slots, (T)now_wrapped);     \
    break;                                                                                          \
  }
    case 1: SSPD_AM(uint8_t)
    case 2: SSPD_AM(uint16_t)
    case 4: SSPD_AM(uint32_t)
    case 8: SSPD_AM(uint64_t)
#undef SSPD_AM
    default:
      return SSPD_ERR_CONFIG;
  }
  return check_launch();
}

extern "C" int sspd_route_pairs(const uint32_t* hips, const uint32_t* oips, uint64_t n, const sspd_params* p,
                                const sspd_divisor* n_wp, int mode, uint64_t index_base, int64_t* lanes_out,
                                void* stream) {
  if (!p || !n_wp || n_wp->d < 1 || (mode != 0 && mode != 1)) return SSPD_ERR_CONFIG;
  if (n == 0) return SSPD_OK;
  if (!lanes_out || (mode == 0 && (!hips || !oips))) return SSPD_ERR_DATA;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = grid_for(route_kernel, 256, n);
  route_kernel<<<grid, 256, 0, st>>>(hips, oips, n, p->seed_route, *n_wp, mode, index_base, lanes_out);
  return check_launch();
}
