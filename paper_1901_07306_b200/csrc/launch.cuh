// Launch helpers shared by every translation unit of libsspd_b200.so.
#pragma once
#include <cuda_runtime.h>
#include "sspd_common.cuh"

namespace sspd {

// Persistent-style grid: (resident blocks per SM) x (SM count), capped by the
// work so that tiny batches do not launch idle blocks.  Sized once per
// kernel per device.
// The occupancy answer is cached per kernel instantiation (one process drives
// one device; a benign race at worst recomputes the same value).
template <typename K>
static inline int grid_for(K kernel, int block, uint64_t work_items) {
  static int cached_full = 0;
  static int cached_block = 0;
  if (cached_full == 0 || cached_block != block) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, 0);
    if (per_sm < 1) per_sm = 1;
    cached_block = block;
    cached_full = sms * per_sm;
  }
  uint64_t full = (uint64_t)cached_full;
  uint64_t need = (work_items + block - 1) / block;
  if (need < 1) need = 1;
  return (int)(need < full ? need : full);
}

static inline int check_launch() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SSPD_OK : SSPD_ERR_CUDA;
}

// Geometry the kernels implement (SURVEY.md §8b "reject geometry outside
// what the kernels implement").  The host layer validates the reference
// constraints (short_sketch.py:135-181) before building the block.
static inline int validate_params(const sspd_params* p) {
  if (!p) return SSPD_ERR_CONFIG;
  if (p->sr < 2 || p->sr > SSPD_MAX_SR) return SSPD_ERR_CONFIG;
  if (p->lr < 1 || p->lr > SSPD_MAX_LR) return SSPD_ERR_CONFIG;
  if (p->r > 16 || p->lp_bits < 1 || p->lp_bits > 32) return SSPD_ERR_CONFIG;
  if (p->g < 1 || p->g > 64) return SSPD_ERR_CONFIG;
  if (!(p->reg_bytes == 1 || p->reg_bytes == 2 || p->reg_bytes == 4 || p->reg_bytes == 8)) return SSPD_ERR_CONFIG;
  if (p->k < 8 || (p->k & 7u) || p->lc < 1) return SSPD_ERR_CONFIG;
  if (p->div_k.d != p->k || p->div_lc.d != p->lc || p->div_g.d != p->g) return SSPD_ERR_CONFIG;
  for (uint32_t i = 0; i < p->sr; ++i) {
    if (p->ibn[i] < 1 || p->ibn[i] > p->lp_bits || p->ibn[i] > 16) return SSPD_ERR_CONFIG;
    if (p->isb[i] >= p->lp_bits) return SSPD_ERR_CONFIG;
    if (p->sc[i] != (1u << p->ibn[i])) return SSPD_ERR_CONFIG;
  }
  return SSPD_OK;
}

// K1b (scan_bpart.cu): the LDCA cut along its b axis, one 16-B entry per
// packet; preferred whenever its plan applies.  `slide` (optional): the
// sliding SEAV sink -- u16 stamps (+ view, slot log) of the sampled packets
// instead of SEAV bits.
struct SlideSeavSink {
  uint16_t* pool;
  uint32_t now;
  uint32_t* view;
  uint32_t* log;
  unsigned long long* log_head;
  uint32_t log_mask;
};
uint64_t scan_bpart_scratch(const sspd_params* p, uint64_t chunk);
int scan_bpart_launch(const uint32_t* hips, const uint32_t* oips, uint64_t n, const sspd_params* p, uint8_t* seav,
                      uint8_t* ldca, void* scratch, uint64_t scratch_bytes, uint64_t chunk, void* stream,
                      bool dst_zero = false, const SlideSeavSink* slide = nullptr);

}  // namespace sspd
