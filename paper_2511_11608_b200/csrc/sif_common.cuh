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
  uint32_t p = 0;
#pragma unroll
  for (int i = 31; i >= 0; --i) {
    p ^= b & (0u - ((a >> i) & 1u));
    b = (b >> 1) ^ (kCrcPoly & (0u - (b & 1u)));
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
// kPieceShift[j] = x^(8 * CRC_PIECE * j) mod P: shifts a piece's raw CRC over j whole
// pieces (pieces are aligned to the end of the CRC range).  Filled by the host
// (sif_lib.cu, crc_tables_init) before the first CRC launch.
constexpr uint64_t CRC_PIECE = 2048;      // bytes per warp-level CRC piece (64 per lane)
constexpr int CRC_PIECES_MAX = 65536;     // payloads up to 128 MiB
__device__ uint32_t kPieceShift[CRC_PIECES_MAX];

// Raw CRC-32 of bytes [e0, e1) (0 < e1 - e0 <= CRC_PIECE) of a 4-byte aligned buffer,
// shifted to e1, computed by one warp (all lanes call; result in every lane).  Lane l
// owns the 64 bytes ending 64*(31-l) bytes before e1; bytes before e0 are taken as zero
// (leading zeros do not change a raw CRC).  stage: >= 544 words of this warp's shared
// memory; t4: kCrcTab4 in shared memory.
template <bool GENERIC = false>
__device__ __forceinline__ uint32_t crc_piece_warp(const uint8_t* base, uint64_t e0, uint64_t e1, const uint32_t* t4,
                                                   uint32_t* stage) {
  const int lane = threadIdx.x & 31;
  const int64_t rs = (int64_t)e1 - (int64_t)CRC_PIECE;  // byte address of the piece start
  const int64_t fl = rs >= 0 ? rs / 4 : -((-rs + 3) / 4);
  const uint32_t sh8 = (uint32_t)(rs - 4 * fl) * 8u;
  const uint32_t* gw = reinterpret_cast<const uint32_t*>(base);
  const int64_t w_lo = (int64_t)(e0 / 4), w_hi = (int64_t)((e1 + 3) / 4);  // words holding [e0, e1)
#pragma unroll
  for (int k = 0; k < 17; ++k) {
    const int j = lane + 32 * k;
    const int64_t wi = fl + j;
    stage[j] = (wi >= w_lo && wi < w_hi) ? (GENERIC ? gw[wi] : __ldcg(gw + wi)) : 0u;
  }
  __syncwarp();
  uint32_t c = 0;
#pragma unroll 4
  for (int k = 0; k < 16; ++k) {
    const int j = 16 * lane + k;
    uint32_t v = sh8 ? __funnelshift_r(stage[j], stage[j + 1], sh8) : stage[j];
    const int64_t a = rs + 4 * (int64_t)j;
    if (a + 4 <= (int64_t)e0) v = 0;
    else if (a < (int64_t)e0) v &= 0xFFFFFFFFu << (8u * (uint32_t)((int64_t)e0 - a));
    const uint32_t x = v ^ c;
    c = t4[768 + (x & 0xFFu)] ^ t4[512 + ((x >> 8) & 0xFFu)] ^ t4[256 + ((x >> 16) & 0xFFu)] ^ t4[x >> 24];
  }
  __syncwarp();
  if (c) c = crc_mult(kCrcShift64[31 - lane], c);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c ^= __shfl_xor_sync(0xFFFFFFFFu, c, o);
  return c;
}

// Raw CRC of [b0, b1) by the warps of a CTA of NT threads: one 2 KiB piece per warp per
// round (pieces aligned to b1, combined with kPieceShift), so a short range (a token's
// payload) costs one warp-piece instead of NT*64 staged bytes.  Result in every thread.
// stage: >= 544 words per warp; red: >= NT/32 words.  GENERIC: base may be shared memory.
template <int NT, bool GENERIC = false>
__device__ uint32_t crc_cta_pieces(const uint8_t* base, uint64_t b0, uint64_t b1, const uint32_t* t4, uint32_t* red,
                                   uint32_t* stage) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t n = b1 > b0 ? b1 - b0 : 0;
  const uint32_t np = (uint32_t)((n + CRC_PIECE - 1) / CRC_PIECE);
  uint32_t acc = 0;
  for (uint32_t piece = (uint32_t)w; piece < np; piece += NW) {
    const uint64_t e1 = b1 - (uint64_t)piece * CRC_PIECE;
    const uint64_t e0 = e1 - b0 > CRC_PIECE ? e1 - CRC_PIECE : b0;
    const uint32_t raw = crc_piece_warp<GENERIC>(base, e0, e1, t4, stage + w * 544);
    if (raw) acc ^= piece ? crc_mult(kPieceShift[piece], raw) : raw;
  }
  if (lane == 0) red[w] = acc;
  __syncthreads();
  uint32_t tot = 0;
#pragma unroll
  for (int k = 0; k < NW; ++k) tot ^= red[k];
  __syncthreads();
  return tot;
}

__device__ __forceinline__ uint32_t crc_finish(uint32_t raw_total, uint64_t len) {
  return raw_total ^ crc_mult(crc_x8n(len), 0xFFFFFFFFu) ^ 0xFFFFFFFFu;
}
// Raw CRC of bytes [b0, b1) of a 4-byte aligned buffer (read through L2), slice-by-4.
// t4 = 4 x 256 table in shared memory (kCrcTab4).
__device__ __forceinline__ uint32_t crc_raw_range(const uint8_t* base, uint64_t b0, uint64_t b1,
                                                  const uint32_t* t4) {
  uint32_t c = 0;
  if (b0 >= b1) return 0;
  const uint32_t* w = reinterpret_cast<const uint32_t*>(base);
  uint64_t i = b0;
  while (i < b1 && (i & 3u)) {
    const uint32_t byte = (__ldcg(w + (i >> 2)) >> (8u * (uint32_t)(i & 3u))) & 0xFFu;
    c = t4[(c ^ byte) & 0xFFu] ^ (c >> 8);
    ++i;
  }
  while (i + 4 <= b1) {
    const uint32_t x = __ldcg(w + (i >> 2)) ^ c;
    c = t4[768 + (x & 0xFFu)] ^ t4[512 + ((x >> 8) & 0xFFu)] ^ t4[256 + ((x >> 16) & 0xFFu)] ^ t4[x >> 24];
    i += 4;
  }
  if (i < b1) {
    const uint32_t word = __ldcg(w + (i >> 2));
    while (i < b1) {
      const uint32_t byte = (word >> (8u * (uint32_t)(i & 3u))) & 0xFFu;
      c = t4[(c ^ byte) & 0xFFu] ^ (c >> 8);
      ++i;
    }
  }
  return c;
}
// Raw CRC of [b0, b1) computed by all NT threads of a CTA.  256-byte chunks are aligned to
// b1 so each combine level uses a constant multiplier x^(8*256*2^k) = kX2n[11+k] (leading
// zero bytes do not change a raw CRC, so the partial first chunk needs no special case).
// Result returned in every thread.  red: >= NT/32 + 1 u32 of shared memory.
template <int NT>
__device__ uint32_t crc_cta_raw(const uint8_t* base, uint64_t b0, uint64_t b1, const uint32_t* t4, uint32_t* red) {
  constexpr int NW = NT / 32;
  constexpr int LOGNW = NW >= 16 ? 4 : NW >= 8 ? 3 : NW >= 4 ? 2 : NW >= 2 ? 1 : 0;
  constexpr uint64_t L = 256;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint64_t n = b1 > b0 ? b1 - b0 : 0;
  const uint64_t span = L * NT;
  const int64_t rounds = (int64_t)((n + span - 1) / span);
  uint32_t total = 0;
  for (int64_t q = rounds - 1; q >= 0; --q) {
    const int64_t rs = (int64_t)b1 - (int64_t)span * (q + 1);
    int64_t c0 = rs + (int64_t)L * tid, c1 = c0 + (int64_t)L;
    if (c0 < (int64_t)b0) c0 = (int64_t)b0;
    uint32_t c = c1 > c0 ? crc_raw_range(base, (uint64_t)c0, (uint64_t)c1, t4) : 0u;
#pragma unroll 1
    for (int k = 0; k < 5; ++k) {
      const uint32_t v2 = __shfl_down_sync(0xFFFFFFFFu, c, 1 << k);
      if ((lane & ((2 << k) - 1)) == 0) c = crc_mult(c, kX2n[11 + k]) ^ v2;
    }
    if (lane == 0) red[wid] = c;
    __syncthreads();
    if (wid == 0) {
      c = lane < NW ? red[lane] : 0u;
#pragma unroll 1
      for (int k = 0; k < LOGNW; ++k) {
        const uint32_t v2 = __shfl_down_sync(0xFFFFFFFFu, c, 1 << k);
        if ((lane & ((2 << k) - 1)) == 0) c = crc_mult(c, kX2n[16 + k]) ^ v2;
      }
      if (lane == 0) total = crc_mult(total, kX2n[11 + 5 + LOGNW]) ^ c;
    }
    __syncthreads();
  }
  if (tid == 0) red[NW] = total;
  __syncthreads();
  const uint32_t r = red[NW];
  __syncthreads();
  return r;
}

// Raw CRC of [b0, b1) by all NT threads.  Each round of 64*NT bytes (aligned to b1) is
// staged into shared memory with coalesced loads; every thread CRCs one 64-byte chunk and
// shifts it to the round end with one multiply by kCrcShift64[NT-1-t] (independent across
// threads), then an XOR reduction; rounds combine with x^(8*64*NT) = kX2n[9 + log2 NT].
// stage: >= 16*NT u32 of shared memory; red: >= NT/32 + 1 u32.
// part/nparts: this CTA handles rounds q = part, part + nparts, ... (counted from b1) and
// returns its partial already shifted to b1; partials of all parts XOR to the raw CRC.
// GENERIC: base is any 4-byte aligned address (e.g. a shared-memory copy of the bytes),
// read with plain loads; otherwise global memory read through L2 (ld.global.cg).
template <int NT, bool GENERIC = false>
__device__ uint32_t crc_cta_staged(const uint8_t* base, uint64_t b0, uint64_t b1, const uint32_t* t4, uint32_t* red,
                                   uint32_t* stage, uint32_t part = 0, uint32_t nparts = 1) {
  constexpr int NW = NT / 32;
  constexpr int LOGNT = NT >= 1024 ? 10 : NT >= 512 ? 9 : NT >= 256 ? 8 : NT >= 128 ? 7 : NT >= 64 ? 6 : 5;
  static_assert(NT <= 1024, "crc_cta_staged: at most 1024 threads");
  constexpr int64_t L = 64, SPAN = L * NT, WORDS = SPAN / 4;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint64_t n = b1 > b0 ? b1 - b0 : 0;
  const int64_t rounds = (int64_t)((n + SPAN - 1) / SPAN);
  const uint32_t* gw = reinterpret_cast<const uint32_t*>(base);
  // x^(8*64*(NT-1-tid)): the table covers 512 chunks; x^(8*64*512) = x^(2^18) = kX2n[18]
  const uint32_t myshift = (NT - 1 - tid) < 512 ? kCrcShift64[NT - 1 - tid]
                                                : crc_mult(kCrcShift64[NT - 1 - tid - 512], kX2n[18]);
  const int lognp = nparts >= 8 ? 3 : nparts >= 4 ? 2 : nparts >= 2 ? 1 : 0;
  uint32_t total = 0;
  int64_t qtop = rounds - 1;
  while (qtop >= 0 && (uint64_t)qtop % nparts != part) --qtop;
  for (int64_t q = qtop; q >= 0; q -= nparts) {
    const int64_t rs = (int64_t)b1 - SPAN * (q + 1);  // byte address of stage[0]
    const int64_t fl = rs >= 0 ? rs / 4 : -((-rs + 3) / 4);
    const uint32_t sh8 = (uint32_t)(rs - 4 * fl) * 8u;
    // 16 words per thread, loads issued together (one memory round trip per round)
    uint32_t lov[WORDS / NT], hiv[WORDS / NT];
#pragma unroll
    for (int k = 0; k < WORDS / NT; ++k) {
      const int64_t j = tid + (int64_t)k * NT;
      const int64_t a = rs + 4 * j;
      const int64_t w0 = fl + j;
      if (GENERIC) {
        lov[k] = (a + 4 > (int64_t)b0 && w0 >= 0 && 4 * w0 + 4 > (int64_t)b0) ? gw[w0] : 0u;
        hiv[k] = (a + 4 > (int64_t)b0 && sh8 && 4 * (w0 + 1) < (int64_t)b1) ? gw[w0 + 1] : 0u;
      } else {
        lov[k] = (a + 4 > (int64_t)b0 && w0 >= 0 && 4 * w0 + 4 > (int64_t)b0) ? __ldcg(gw + w0) : 0u;
        hiv[k] = (a + 4 > (int64_t)b0 && sh8 && 4 * (w0 + 1) < (int64_t)b1) ? __ldcg(gw + w0 + 1) : 0u;
      }
    }
#pragma unroll
    for (int k = 0; k < WORDS / NT; ++k) {
      const int64_t j = tid + (int64_t)k * NT;
      const int64_t a = rs + 4 * j;
      uint32_t v = sh8 ? __funnelshift_r(lov[k], hiv[k], sh8) : lov[k];
      if (a + 4 <= (int64_t)b0) v = 0;
      else if (a < (int64_t)b0) v &= 0xFFFFFFFFu << (8u * (uint32_t)((int64_t)b0 - a));
      stage[j] = v;
    }
    __syncthreads();
    uint32_t c = 0;
    if (rs + L * (tid + 1) > (int64_t)b0) {  // a chunk wholly before b0 is zeros: raw CRC 0
      const uint32_t* w = stage + tid * (L / 4);
#pragma unroll 4
      for (int k = 0; k < L / 4; ++k) {
        const uint32_t x = w[k] ^ c;
        c = t4[768 + (x & 0xFFu)] ^ t4[512 + ((x >> 8) & 0xFFu)] ^ t4[256 + ((x >> 16) & 0xFFu)] ^ t4[x >> 24];
      }
      if (c) c = crc_mult(myshift, c);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c ^= __shfl_xor_sync(0xFFFFFFFFu, c, o);
    if (lane == 0) red[wid] = c;
    __syncthreads();
    if (tid == 0) {
      uint32_t rq = 0;
      for (int k = 0; k < NW; ++k) rq ^= red[k];
      total = crc_mult(total, kX2n[9 + LOGNT + lognp]) ^ rq;
    }
    __syncthreads();
  }
  if (tid == 0) {
    // shift this part's rounds (q = part + k*nparts) down by part rounds
    for (int k = 0; k < 4; ++k)
      if ((part >> k) & 1u) total = crc_mult(total, kX2n[9 + LOGNT + k]);
    red[NW] = total;
  }
  __syncthreads();
  const uint32_t r = red[NW];
  __syncthreads();
  return r;
}

// Walks the IF owning consecutive global piece numbers gp of a prefix table base[0..n]
// (pieces of IF i are base[i] .. base[i+1]-1): one binary search for the first piece of a
// warp's contiguous range, then forward steps (no dependent-load chain per piece).
struct PieceWalk {
  const uint32_t* base;
  int n, i;
  uint32_t b0, b1;
  __device__ __forceinline__ void init(const uint32_t* bs, int nn) { base = bs; n = nn; i = -1; b0 = b1 = 0; }
  __device__ __forceinline__ int at(uint64_t gp) {
    if (i < 0) {
      int lo = 0, hi = n - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (base[mid] <= gp) lo = mid; else hi = mid - 1;
      }
      i = lo;
      b0 = base[i];
      b1 = base[i + 1];
    }
    while (gp >= b1) {
      ++i;
      b0 = b1;
      b1 = base[i + 1];
    }
    return i;
  }
};

// ---------------------------------------------------------------- bulk-async copies
// cp.async.bulk (the TMA engine, non-tensor form) global -> shared, completing on an
// mbarrier: one thread issues the copy, every thread waits on the barrier's phase.
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// bytes % 16 == 0, dst / src 16-byte aligned; arrives on `bar` expecting the bytes
__device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// Fast exact u32 division / modulo by an invariant divisor (Lemire fastmod, 64-bit M).
struct FastDiv {
  uint64_t M;
  uint32_t d;
  __host__ __device__ void init(uint32_t dd) {
    d = dd;
    M = dd ? (~0ull / dd + 1ull) : 0ull;
  }
  __device__ __forceinline__ uint32_t div(uint32_t x) const { return d == 1 ? x : (uint32_t)__umul64hi(M, (uint64_t)x); }
  __device__ __forceinline__ uint32_t mod(uint32_t x) const {
    return d == 1 ? 0u : (uint32_t)__umul64hi(M * (uint64_t)x, (uint64_t)d);
  }
};

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
__device__ __forceinline__ uint32_t warp_incl_scan_u32(uint32_t x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

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

// Block-wide exclusive scan of a u32; total in *total.  scratch >= 33 u32 in smem.
__device__ __forceinline__ uint32_t block_excl_scan_u32(uint32_t v, uint32_t* scratch, uint32_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) scratch[wid] = x;
  __syncthreads();
  if (wid == 0) {
    const uint32_t t = lane < nw ? scratch[lane] : 0u;
    uint32_t s = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) scratch[lane] = s - t;
    if (lane == 31) scratch[32] = s;
  }
  __syncthreads();
  const uint32_t r = scratch[wid] + x - v;
  *total = scratch[32];
  __syncthreads();
  return r;
}

}  // namespace sif
