// SURVEY.md §8(f) "next" rows on the device:
//   * trace ingest -- the reference's 12-byte (slice, hip, oip) records
//     (evaluation.py:21, read_trace :235-254) unpacked to the SoA layout the
//     scan kernels stream;
//   * frame checksum -- CRC-32 (the zlib.crc32 of distributed.py:100,
//     :121-123) of a device payload, so watch-point frames can be sealed and
//     checked straight from HBM.
//
// CRC-32 here is the reflected IEEE polynomial 0xEDB88320 with the usual
// ~ conditioning (zlib).  The payload is cut into fixed chunks; one thread
// computes each chunk's CRC with a slice-by-8 table in shared memory, and
// a single CTA folds the chunk CRCs pairwise with the GF(2) combination
// crc(A||B) = (crc(A) * x^(8|B|) mod P) xor crc(B) -- the algebra behind
// zlib's crc32_combine, restated for the device.
#include <cuda_runtime.h>
#include "sspd_common.cuh"
#include "launch.cuh"

namespace sspd {

constexpr uint32_t kCrcPoly = 0xEDB88320u;
constexpr uint32_t kCrcChunk = 4096;  // bytes per thread in the chunk pass

// ------------------------------------------------------------ unpack
__global__ void __launch_bounds__(256) unpack_records_kernel(const uint32_t* __restrict__ rec, uint64_t n,
                                                             uint32_t* slices, uint32_t* hips, uint32_t* oips) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
    const uint32_t* r = rec + 3 * j;  // little-endian <u4 fields
    const uint32_t s = __ldcs(r), h = __ldcs(r + 1), o = __ldcs(r + 2);
    if (slices) slices[j] = s;
    hips[j] = h;
    oips[j] = o;
  }
}

// ------------------------------------------------------------- CRC-32
__device__ __forceinline__ uint32_t gf2_mulmod(uint32_t a, uint32_t b) {
  // a * b mod P in the reflected representation (bit 31 = x^0)
  uint32_t m = 1u << 31, prod = 0;
  for (int i = 0; i < 32; ++i) {
    if (a & m) prod ^= b;
    m >>= 1;
    b = (b & 1u) ? (b >> 1) ^ kCrcPoly : (b >> 1);
  }
  return prod;
}

// x^(8 n) mod P, from the table pow2[k] = x^(2^k) mod P
__device__ uint32_t x8n_mod(uint64_t n, const uint32_t* pow2) {
  uint32_t acc = 1u << 31;  // x^0
  uint32_t k = 3;           // 8 n = n << 3
  while (n) {
    if (n & 1) acc = gf2_mulmod(pow2[k & 63], acc);
    n >>= 1;
    ++k;
  }
  return acc;
}

__global__ void __launch_bounds__(256) crc_chunks_kernel(const uint8_t* __restrict__ data, uint64_t n,
                                                         uint32_t* chunk_crc, uint64_t nchunks) {
  __shared__ uint32_t tab[8][256];
  for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) {
    uint32_t c = i;
    for (int b = 0; b < 8; ++b) c = (c & 1u) ? (c >> 1) ^ kCrcPoly : (c >> 1);
    tab[0][i] = c;
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x)
    for (int t = 1; t < 8; ++t) tab[t][i] = (tab[t - 1][i] >> 8) ^ tab[0][tab[t - 1][i] & 0xFFu];
  __syncthreads();
  const uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  const uint64_t lo = c * kCrcChunk, hi = min(n, lo + kCrcChunk);
  uint32_t crc = 0xFFFFFFFFu;
  uint64_t i = lo;
  if (((reinterpret_cast<uintptr_t>(data) + lo) & 7u) == 0) {  // slice-by-8 over aligned 8-byte words
    for (; i + 8 <= hi; i += 8) {
      const uint2 w = *reinterpret_cast<const uint2*>(data + i);
      const uint32_t x = w.x ^ crc, y = w.y;
      crc = tab[7][x & 0xFFu] ^ tab[6][(x >> 8) & 0xFFu] ^ tab[5][(x >> 16) & 0xFFu] ^ tab[4][x >> 24] ^
            tab[3][y & 0xFFu] ^ tab[2][(y >> 8) & 0xFFu] ^ tab[1][(y >> 16) & 0xFFu] ^ tab[0][y >> 24];
    }
  }
  for (; i < hi; ++i) crc = (crc >> 8) ^ tab[0][(crc ^ data[i]) & 0xFFu];
  chunk_crc[c] = crc ^ 0xFFFFFFFFu;
}

// One CTA folds the chunk CRCs: level by level, crc(L||R) = crc(L)*x^(8|R|) ^ crc(R).
__global__ void __launch_bounds__(1024) crc_fold_kernel(uint32_t* crc, uint64_t nchunks, uint64_t n,
                                                        uint32_t* out) {
  __shared__ uint32_t pow2[64];
  if (threadIdx.x == 0) {
    uint32_t p = 1u << 30;  // x^1
    for (int k = 0; k < 64; ++k) {
      pow2[k] = p;
      p = gf2_mulmod(p, p);
    }
  }
  __syncthreads();
  // span = chunks per node at this level; only the last node can be short
  for (uint64_t span = 1; span < nchunks; span <<= 1) {
    for (uint64_t left = threadIdx.x * 2 * span; left < nchunks; left += (uint64_t)blockDim.x * 2 * span) {
      const uint64_t right = left + span;
      if (right >= nchunks) continue;
      const uint64_t rlo = right * kCrcChunk;
      const uint64_t rhi = min(n, (right + span) * kCrcChunk);
      crc[left] = gf2_mulmod(x8n_mod(rhi - rlo, pow2), crc[left]) ^ crc[right];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = nchunks ? crc[0] : 0u;
}

}  // namespace sspd

using namespace sspd;

extern "C" int sspd_unpack_records(const uint8_t* records, uint64_t n, uint32_t* slices, uint32_t* hips,
                                   uint32_t* oips, void* stream) {
  if (n == 0) return SSPD_OK;
  if (!records || !hips || !oips || (reinterpret_cast<uintptr_t>(records) & 3u)) return SSPD_ERR_DATA;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = grid_for(unpack_records_kernel, 256, n);
  unpack_records_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const uint32_t*>(records), n, slices, hips, oips);
  return check_launch();
}

extern "C" int sspd_crc32(const uint8_t* data, uint64_t n, uint32_t* out, void* scratch, uint64_t* scratch_bytes,
                          void* stream) {
  if (!scratch_bytes) return SSPD_ERR_DATA;
  const uint64_t nchunks = (n + kCrcChunk - 1) / kCrcChunk;
  const uint64_t need = 4 * (nchunks ? nchunks : 1);
  if (!scratch) {  // size query
    *scratch_bytes = need;
    return SSPD_OK;
  }
  if (!out) return SSPD_ERR_DATA;
  if (*scratch_bytes < need) return SSPD_ERR_CAPACITY;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint32_t* chunk_crc = static_cast<uint32_t*>(scratch);
  if (nchunks) {
    if (!data) return SSPD_ERR_DATA;
    crc_chunks_kernel<<<(unsigned)((nchunks + 255) / 256), 256, 0, st>>>(data, n, chunk_crc, nchunks);
  }
  crc_fold_kernel<<<1, 1024, 0, st>>>(chunk_crc, nchunks, n, out);
  return check_launch();
}
