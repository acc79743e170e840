// Shared device helpers for the B200 SLICER IF codec kernels (sm_100a).
//
// Bit-exactness notes:
//  * every float64 op that the reference evaluates with NumPy (atkf.py:31-34, :72-73,
//    quant.py:59-62, :71-73) is written with explicit __d*_rn intrinsics so nvcc cannot
//    contract a*b+c into an FMA;
//  * tie-break keys are splitmix64 of the flat index (rng.py:60-68);
//  * the wire format is a big-endian bit stream (bitstream.py:12-20): MSB-first within
//    bytes, so a little-endian u32 load is byte-swapped with PRMT before bit extraction.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "sif.h"
#include "sif_crc_tables.cuh"

namespace sif {

namespace cg = cooperative_groups;

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr int kHeaderBytes = 32;     // codec.py:51
constexpr int kBlockMetaBytes = 13;  // codec.py:52
constexpr int kCrcBytes = 4;         // codec.py:53
constexpr int kQMax = 16;            // quant.py:21
constexpr uint32_t kNonFiniteKey = 0x7F800000u;

// ---------------------------------------------------------------- hashing (rng.py:23-27)
__device__ __forceinline__ uint64_t splitmix(uint64_t seed, uint64_t i) {
  uint64_t z = seed + (i + 1ull) * kGolden;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// codec.py:57-58: max(1, (k-1).bit_length()); k == 0 gives (-1).bit_length() == 1.
__host__ __device__ __forceinline__ uint32_t col_bits(uint32_t k) {
  if (k <= 2u) return 1u;
  uint32_t v = k - 1u, b = 0;
  while (v) { ++b; v >>= 1; }
  return b;
}

// atkf.py:31-34: int(floor((1.0 - s) * t + 1e-9)), no FMA contraction.
__host__ __device__ __forceinline__ uint64_t keep_count(double s, uint64_t t) {
#ifdef __CUDA_ARCH__
  double v = __dadd_rn(__dmul_rn(__dsub_rn(1.0, s), (double)t), 1e-9);
#else
  volatile double a = 1.0 - s;
  volatile double b = a * (double)t;
  double v = b + 1e-9;
#endif
  double f = floor(v);
  return f <= 0.0 ? 0ull : (uint64_t)f;
}

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// ---------------------------------------------------------------- CRC-32 (zlib.crc32)
// Reflected GF(2) arithmetic: raw CRC (init 0, no xor-out) is linear, so chunk CRCs
// combine as raw(A||B) = raw(A)*x^(8|B|) ^ raw(B) and
// zlib.crc32(m) = raw(m) ^ (0xFFFFFFFF * x^(8|m|)) ^ 0xFFFFFFFF.
__device__ __forceinline__ uint32_t crc_mult(uint32_t a, uint32_t b) {
  uint32_t m = 1u << 31, p = 0;
  for (;;) {
    if (a & m) {
      p ^= b;
      if ((a & (m - 1u)) == 0) break;
    }
    m >>= 1;
    b = (b & 1u) ? (b >> 1) ^ kCrcPoly : b >> 1;
  }
  return p;
}
__device__ __forceinline__ uint32_t crc_x8n(uint64_t nbytes) {
  uint32_t p = 1u << 31;
  int k = 3;
  while (nbytes) {
    if (nbytes & 1ull) p = crc_mult(kX2n[k & 63], p);
    nbytes >>= 1;
    ++k;
  }
  return p;
}
__device__ __forceinline__ uint32_t crc_shift(uint32_t c, uint64_t nbytes) {
  return c ? crc_mult(crc_x8n(nbytes), c) : 0u;
}
__device__ __forceinline__ uint32_t crc_finish(uint32_t raw_total, uint64_t len) {
  return raw_total ^ crc_mult(crc_x8n(len), 0xFFFFFFFFu) ^ 0xFFFFFFFFu;
}
// Raw CRC of bytes [b0, b1) of a 4-byte aligned buffer, read through L2 (ld.global.cg).
__device__ __forceinline__ uint32_t crc_raw_range(const uint8_t* base, uint64_t b0, uint64_t b1,
                                                  const uint32_t* tab) {
  uint32_t c = 0;
  if (b0 >= b1) return 0;
  const uint32_t* w = reinterpret_cast<const uint32_t*>(base);
  uint64_t i = b0;
  uint32_t word = __ldcg(w + (i >> 2));
  while (i < b1) {
    if ((i & 3u) == 0u && i + 4 <= b1) {
      word = __ldcg(w + (i >> 2));
      c = tab[(c ^ word) & 0xFFu] ^ (c >> 8);
      c = tab[(c ^ (word >> 8)) & 0xFFu] ^ (c >> 8);
      c = tab[(c ^ (word >> 16)) & 0xFFu] ^ (c >> 8);
      c = tab[(c ^ (word >> 24)) & 0xFFu] ^ (c >> 8);
      i += 4;
      continue;
    }
    if ((i & 3u) == 0u || i == b0) word = __ldcg(w + (i >> 2));
    uint32_t byte = (word >> (8u * (uint32_t)(i & 3u))) & 0xFFu;
    c = tab[(c ^ byte) & 0xFFu] ^ (c >> 8);
    ++i;
  }
  return c;
}

// ---------------------------------------------------------------- byte stream helpers
// Unaligned little-endian u32 read from a 4-byte aligned buffer.
__device__ __forceinline__ uint32_t ld_u32_le(const uint8_t* base, uint64_t off) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(base);
  uint64_t wi = off >> 2;
  uint32_t sh = 8u * (uint32_t)(off & 3u);
  uint32_t lo = __ldg(w + wi);
  if (sh == 0) return lo;
  uint32_t hi = __ldg(w + wi + 1);
  return __funnelshift_r(lo, hi, sh);
}
__device__ __forceinline__ uint8_t ld_u8(const uint8_t* base, uint64_t off) { return __ldg(base + off); }

// Extract a w-bit MSB-first field at absolute bit offset `bit` (w <= 32).
__device__ __forceinline__ uint32_t ld_field(const uint8_t* base, uint64_t bit, uint32_t w) {
  const uint32_t* p = reinterpret_cast<const uint32_t*>(base);
  uint64_t wi = bit >> 5;
  uint32_t sh = (uint32_t)(bit & 31u);
  uint64_t hi = (uint64_t)bswap32(__ldg(p + wi)) << 32;
  if (sh + w > 32u) hi |= bswap32(__ldg(p + wi + 1));
  uint64_t v = hi << sh;
  return (uint32_t)(v >> (64u - w));
}

__device__ __forceinline__ void st_u32_le_bytes(uint8_t* base, uint64_t off, uint32_t v) {
  base[off] = (uint8_t)v;
  base[off + 1] = (uint8_t)(v >> 8);
  base[off + 2] = (uint8_t)(v >> 16);
  base[off + 3] = (uint8_t)(v >> 24);
}

// ---------------------------------------------------------------- reductions
__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}
__device__ __forceinline__ uint32_t warp_xor(uint32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v ^= __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}

// Block-wide exclusive scan of a u64 (fields packed by the caller); returns the
// exclusive prefix, writes the block total to *total.  `scratch` >= 33 u64 in smem.
__device__ __forceinline__ uint64_t block_excl_scan_u64(uint64_t v, uint64_t* scratch,
                                                        uint64_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) scratch[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint64_t t = lane < nw ? scratch[lane] : 0ull;
    uint64_t s = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint64_t y = __shfl_up_sync(0xFFFFFFFFu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) scratch[lane] = s - t;
    if (lane == nw - 1) scratch[32] = s;
  }
  __syncthreads();
  uint64_t r = scratch[wid] + x - v;
  *total = scratch[32];
  __syncthreads();
  return r;
}

}  // namespace sif
