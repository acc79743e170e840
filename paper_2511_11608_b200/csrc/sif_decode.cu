// sif_decode.cu -- B200 (sm_100a) decoder for the SLICER .sif wire format.
//
// Two launches per batch:
//   sif_parse_kernel   one thread per stream walks the header/block framing exactly in the
//                      order of deserialize (codec.py:320-385) and writes a block table.
//   sif_scatter_kernel one CTA per (stream, row slab): CRC-32 of a payload chunk (combined
//                      with GF(2) shifts), row_ptr/cols validation (codec.py:235-251),
//                      fused unpack + float64 dequantize (quant.py:67-73) + scatter-add
//                      into a float64 shared-memory tile, rounded to fp32 (codec.py:266)
//                      and written once with coalesced stores.  The last CTA of a stream
//                      folds CRC, framing and validation flags into the reference's error
//                      precedence and resets the per-stream accumulators.

#include <stdint.h>

#include "sif_common.cuh"

namespace sif {

constexpr int DNT = 256;
constexpr int TROW_U32 = 16;  // table row: 16 x u32 = 64 bytes
constexpr uint32_t FLAG_CORRUPT = 1u, FLAG_NONFINITE = 2u;

struct DecTile {
  uint32_t ifi, ti, nt, r0, r1, c0, c1, pad;
};

struct DecArgs {
  const sif_dec_desc* descs;
  int n;
  uint32_t* table;        // per IF: (2 + maxb) rows of TROW_U32
  uint64_t table_stride;  // in u32
  uint32_t* acc;          // per IF: {crc, flags, count, pad}
  const DecTile* tiles;
  int ntiles;
  int parse_only;
  int tile_elems;
  int rpc_cap;
  int32_t* status;
  const uint32_t* tiles_per_if;
};

// ------------------------------------------------------------------------------- parse
__device__ __forceinline__ uint32_t rd_u32(const uint8_t* p, uint64_t o) {
  return (uint32_t)p[o] | ((uint32_t)p[o + 1] << 8) | ((uint32_t)p[o + 2] << 16) | ((uint32_t)p[o + 3] << 24);
}

__global__ void sif_parse_kernel(DecArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const sif_dec_desc d = a.descs[i];
  uint32_t* tab = a.table + (uint64_t)i * a.table_stride;
  const uint8_t* in = d.in;
  const uint64_t len = d.in_len;
  const uint64_t max_rows = a.table_stride / TROW_U32 - 2;
  uint32_t pre = 0, walk = 0, N = 0, K = 0, mp = 0, mm = 0, mode = 0, qb = 0, nb = 0, crc = 0;
  if (len < (uint64_t)(kHeaderBytes + kCrcBytes)) pre = SIF_ERR_STREAM_FORMAT;  // codec.py:321
  else if (in[0] != 'S' || in[1] != 'I' || in[2] != 'F' || in[3] != '1') pre = SIF_ERR_STREAM_FORMAT;
  if (!pre) {
    crc = rd_u32(in, len - 4);
    const uint32_t ver = (uint32_t)in[4] | ((uint32_t)in[5] << 8);
    N = rd_u32(in, 6);
    K = rd_u32(in, 10);
    qb = in[22];
    mode = in[27];
    mp = (uint32_t)in[28] | ((uint32_t)in[29] << 8);
    mm = (uint32_t)in[30] | ((uint32_t)in[31] << 8);
    if (ver != 1) walk = SIF_ERR_STREAM_FORMAT;  // codec.py:331-332
    else if (mode > 1) walk = SIF_ERR_STREAM_FORMAT;  // codec.py:333-334
    else {
      uint64_t pos = kHeaderBytes;
      if (mode == 1) {
        if (len < pos + mp + mm) walk = SIF_ERR_STREAM_FORMAT;  // codec.py:340-341
        pos += mp + mm;
      }
      const uint32_t cb = col_bits(K);
      const uint64_t nblk = (uint64_t)mp + mm;
      for (uint64_t b = 0; b < nblk && !walk; ++b) {
        if (len < pos + kBlockMetaBytes + 4ull * ((uint64_t)N + 1)) { walk = SIF_ERR_STREAM_FORMAT; break; }
        const uint32_t q = in[pos];
        if (q < 1 || q > (uint32_t)kQMax) { walk = SIF_ERR_CORRUPT_STREAM; break; }  // codec.py:351-352
        const uint32_t o = rd_u32(in, pos + 1), vmin = rd_u32(in, pos + 5), nnz = rd_u32(in, pos + 9);
        const uint64_t rp = pos + kBlockMetaBytes;
        pos = rp + 4ull * ((uint64_t)N + 1);
        const uint64_t cbytes = ((uint64_t)nnz * cb + 7) / 8, qbytes = ((uint64_t)nnz * q + 7) / 8;
        if (len - kCrcBytes < pos + cbytes + qbytes) { walk = SIF_ERR_STREAM_FORMAT; break; }  // :358
        if (b >= max_rows) { walk = SIF_ERR_CAPACITY; break; }
        uint32_t* row = tab + (2 + b) * TROW_U32;
        row[0] = q; row[1] = nnz; row[2] = o; row[3] = vmin;
        row[4] = (uint32_t)rp; row[5] = (uint32_t)(rp >> 32);
        row[6] = (uint32_t)pos; row[7] = (uint32_t)(pos >> 32);
        row[8] = (uint32_t)(pos + cbytes); row[9] = (uint32_t)((pos + cbytes) >> 32);
        pos += cbytes + qbytes;
      }
      if (!walk && pos != len - kCrcBytes) walk = SIF_ERR_STREAM_FORMAT;  // codec.py:384-385
      nb = (uint32_t)nblk;
    }
  }
  tab[0] = walk; tab[1] = N; tab[2] = K; tab[3] = mp; tab[4] = mm; tab[5] = mode; tab[6] = qb; tab[7] = nb;
  tab[TROW_U32 + 0] = pre;
  tab[TROW_U32 + 1] = crc;
  tab[TROW_U32 + 2] = (uint32_t)len;
  tab[TROW_U32 + 3] = (uint32_t)(len >> 32);
}

// ------------------------------------------------------------------------------- scatter
__global__ void __launch_bounds__(DNT, 4) sif_scatter_kernel(DecArgs a) {
  extern __shared__ __align__(16) uint8_t dsm_raw[];
  uint8_t* dsm = dsm_raw;
  __shared__ uint32_t hdr[2 * TROW_U32];
  __shared__ uint32_t red[DNT / 32 + 2];
  __shared__ uint32_t sflags;
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31;
  // CTAs past the tile list compute one stream's CRC-32 each (codec.py:325-327)
  const bool crc_cta = (int)blockIdx.x >= a.ntiles;
  DecTile t;
  if (crc_cta) {
    t.ifi = blockIdx.x - a.ntiles;
    t.ti = 0; t.nt = 0; t.r0 = t.r1 = t.c0 = t.c1 = 0;
  } else {
    t = a.tiles[blockIdx.x];
  }
  const sif_dec_desc d = a.descs[t.ifi];
  const uint32_t* tab = a.table + (uint64_t)t.ifi * a.table_stride;
  if (tid < 2 * TROW_U32) hdr[tid] = tab[tid];
  if (tid == 0) sflags = 0;
  __syncthreads();
  const uint32_t walk = hdr[0], N = hdr[1], K = hdr[2], mp = hdr[3], nb = hdr[7];
  const uint32_t pre = hdr[TROW_U32 + 0];
  const uint64_t len = d.in_len;
  const uint8_t* in = d.in;
  // number of CTAs that report to this stream's accumulator: its tiles + the CRC CTA
  uint32_t ntiles_if = t.nt;

  if (crc_cta) {
    uint32_t* t4 = reinterpret_cast<uint32_t*>(dsm);
    for (int k = tid; k < 1024; k += DNT) t4[k] = (&kCrcTab4[0][0])[k];
    __syncthreads();
    if (!pre) {
      const uint32_t raw = crc_cta_staged<DNT>(in, 4, len - 4, t4, red, t4 + 1024);
      if (tid == 0) a.acc[4ull * t.ifi + 0] = raw;
    }
    ntiles_if = a.tiles_per_if[t.ifi];
  }
  // ---- validate + dequantize + scatter this row slab
  const bool shape_ok = a.parse_only || (N == d.rows && K == d.cols);
  if (!crc_cta && !a.parse_only && !pre && !walk && shape_ok) {
    const uint32_t R = t.r1 - t.r0, Kc = t.c1 - t.c0;
    const uint32_t E = R * Kc;
    double* tile = reinterpret_cast<double*>(dsm);
    uint32_t* bm = reinterpret_cast<uint32_t*>(tile + a.tile_elems);
    const uint32_t bmw = (uint32_t)(a.tile_elems + 31) / 32;
    uint32_t* rpc = bm + 2 * bmw;
    const bool cached = (uint64_t)(R + 1) * nb <= (uint64_t)a.rpc_cap;
    {
      uint4* t4z = reinterpret_cast<uint4*>(tile);
      for (uint32_t k = tid; k < (E + 1) / 2; k += DNT) t4z[k] = make_uint4(0, 0, 0, 0);
      for (uint32_t k = tid; k < 2 * bmw; k += DNT) bm[k] = 0;
    }
    const uint32_t cb = col_bits(K);
    uint32_t fl = 0;
    if (cached) {
      for (uint64_t k = tid; k < (uint64_t)(R + 1) * nb; k += DNT) {
        const uint32_t b = (uint32_t)(k / (R + 1)), rr = (uint32_t)(k % (R + 1));
        const uint32_t* row = tab + (2ull + b) * TROW_U32;
        const uint64_t rpo = (uint64_t)row[4] | ((uint64_t)row[5] << 32);
        rpc[k] = ld_u32_le(in, rpo + 4ull * (t.r0 + rr));
      }
    }
    __syncthreads();
    for (uint32_t b = 0; b < nb; ++b) {
      const uint32_t* row = tab + (2ull + b) * TROW_U32;
      const uint32_t q = row[0], nnz = row[1];
      const double o = (double)__uint_as_float(row[2]), vmin = (double)__uint_as_float(row[3]);
      const uint64_t rpo = (uint64_t)row[4] | ((uint64_t)row[5] << 32);
      const uint64_t cbit = 8ull * ((uint64_t)row[6] | ((uint64_t)row[7] << 32));
      const uint64_t qbit = 8ull * ((uint64_t)row[8] | ((uint64_t)row[9] << 32));
      const int plane = b < mp ? 0 : 1;
      auto rp = [&](uint32_t rr) -> uint32_t {
        return cached ? rpc[(uint64_t)b * (R + 1) + rr] : ld_u32_le(in, rpo + 4ull * (t.r0 + rr));
      };
      // row pointer checks (codec.py:238-241)
      for (uint32_t rr = tid; rr < R; rr += DNT)
        if (rp(rr + 1) < rp(rr)) fl |= FLAG_CORRUPT;
      if (tid == 0) {
        if (t.r0 == 0 && rp(0) != 0) fl |= FLAG_CORRUPT;
        if (t.r1 == N && rp(R) != nnz) fl |= FLAG_CORRUPT;
      }
      const uint32_t elo = rp(0) < nnz ? rp(0) : nnz;
      const uint32_t ehi = rp(R) < nnz ? rp(R) : nnz;
      for (uint32_t e = elo + tid; e < ehi; e += DNT) {
        // row of entry e: last rr with rp(rr) <= e
        uint32_t lo = 0, hi = R - 1;  // answer in [0, R-1]
        while (lo < hi) {
          const uint32_t mid = (lo + hi + 1) >> 1;
          if (rp(mid) <= e) lo = mid; else hi = mid - 1;
        }
        const uint32_t rr = lo;
        const uint32_t col = ld_field(in, cbit + (uint64_t)e * cb, cb);
        if (col >= K) { fl |= FLAG_CORRUPT; continue; }  // codec.py:242-243
        if (e > rp(rr) && ld_field(in, cbit + (uint64_t)(e - 1) * cb, cb) >= col) fl |= FLAG_CORRUPT;  // :244-247
        if (col < t.c0 || col >= t.c1) continue;
        const uint32_t pos = rr * Kc + (col - t.c0);
        const uint32_t old = atomicOr(bm + plane * bmw + (pos >> 5), 1u << (pos & 31));
        if (old & (1u << (pos & 31))) fl |= FLAG_CORRUPT;  // codec.py:248-250 (overlap)
        const uint32_t code = ld_field(in, qbit + (uint64_t)e * q, q);
        const double v = __dadd_rn(__dmul_rn((double)code, o), vmin);
        atomicAdd(tile + pos, plane ? -v : v);
      }
    }
    __syncthreads();
    float* out = d.out;
    const bool vec4 = (K % 4u) == 0 && (t.c0 % 4u) == 0 && (Kc % 4u) == 0 &&
                      (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
    if (vec4) {
      // 4 consecutive columns per thread: 2 x 16-byte smem loads, one 16-byte global store
      const uint32_t kq = Kc / 4, nq = E / 4;
      FastDiv fq;
      fq.init(kq);
      const double2* t2 = reinterpret_cast<const double2*>(tile);
      for (uint32_t q = tid; q < nq; q += DNT) {
        const uint32_t rr = fq.div(q), c4 = q - rr * kq;
        const double2 a = t2[2 * q], b2 = t2[2 * q + 1];
        const float4 f = make_float4(__double2float_rn(a.x), __double2float_rn(a.y), __double2float_rn(b2.x),
                                     __double2float_rn(b2.y));
        if (!(isfinite(f.x) && isfinite(f.y) && isfinite(f.z) && isfinite(f.w))) fl |= FLAG_NONFINITE;
        *reinterpret_cast<float4*>(out + (uint64_t)(t.r0 + rr) * K + t.c0 + 4 * c4) = f;
      }
    } else {
      FastDiv fc;
      fc.init(Kc);
      for (uint32_t k = tid; k < E; k += DNT) {
        const uint32_t rr = fc.div(k), cc = k - rr * Kc;
        const float f = __double2float_rn(tile[k]);
        if (!isfinite(f)) fl |= FLAG_NONFINITE;
        out[(uint64_t)(t.r0 + rr) * K + t.c0 + cc] = f;
      }
    }
    fl = __reduce_or_sync(0xFFFFFFFFu, fl);
    if (lane == 0 && fl) atomicOr(&sflags, fl);
    __syncthreads();
    if (tid == 0 && sflags) atomicOr(a.acc + 4ull * t.ifi + 1, sflags);
  }

  // ---- last CTA of this stream folds everything into the reference error precedence
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(a.acc + 4ull * t.ifi + 2, 1u) == ntiles_if;  // tiles + CRC CTA
  __syncthreads();
  if (s_last && tid == 0) {
    __threadfence();
    uint32_t* acc = a.acc + 4ull * t.ifi;
    const uint32_t crc_raw = *((volatile uint32_t*)(acc + 0));
    const uint32_t flags = atomicAdd(acc + 1, 0u);
    int st = SIF_OK;
    if (pre) st = (int)pre;
    else if (crc_finish(crc_raw, len - 8) != hdr[TROW_U32 + 1]) st = SIF_ERR_STREAM_FORMAT;  // :325-327
    else if (walk) st = (int)walk;
    else if (!shape_ok) st = SIF_ERR_CAPACITY;
    else if (!a.parse_only) {
      if (flags & FLAG_CORRUPT) st = SIF_ERR_CORRUPT_STREAM;
      else if (N < 1 || K < 1) st = SIF_ERR_SHAPE;  // tensor.py:27-28
      else if (flags & FLAG_NONFINITE) st = SIF_ERR_NONFINITE;  // tensor.py:35-36
    }
    a.status[t.ifi] = st;
    acc[0] = 0; acc[1] = 0; acc[2] = 0;
  }
}

}  // namespace sif
