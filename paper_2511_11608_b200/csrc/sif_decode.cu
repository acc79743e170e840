// sif_decode.cu -- B200 (sm_100a) decoder for the SLICER .sif wire format.
//
// Four launches per batch:
//   sif_parse_kernel   one thread per stream walks the header/block framing exactly in the
//                      order of deserialize (codec.py:320-385) and writes a block table.
//   sif_dcrc_kernel    one CTA per 64 KiB CRC-32 segment of a stream (GF(2)-combined).
//   sif_scatter_kernel one warp per work item (a group of rows, or a 4096-column segment):
//                      row_ptr/cols validation (codec.py:235-251), fused unpack + float64
//                      dequantize (quant.py:67-73), fp32 values (codec.py:266) stored in
//                      place into the item's zero-filled output.
//   sif_dfinal_kernel  folds CRC, framing and validation flags into the reference's error
//                      precedence and resets the per-stream accumulators.

#include <stdint.h>

#include "sif_common.cuh"

namespace sif {

constexpr int DNT = 256;
constexpr int TROW_U32 = 16;  // table row: 16 x u32 = 64 bytes
constexpr uint32_t FLAG_CORRUPT = 1u, FLAG_NONFINITE = 2u;
// Failure reasons (table row 1, words 4..8) so the host can raise the reference's message
// (codec.py:320-385, :235-251, tensor.py:27-36); see errors.py REASONS.
enum : uint32_t {
  R_NONE = 0, R_SHORT = 1, R_MAGIC = 2, R_CRC = 3, R_VERSION = 4, R_MODE = 5, R_QVEC = 6, R_BLKHDR = 7,
  R_QRANGE = 8, R_BLKPAY = 9, R_TRAIL = 10, R_CAPACITY = 11, R_SHAPE_MISMATCH = 12, R_LEN_OVER = 13, R_CORRUPT = 16,
  R_SHAPE = 32, R_NONFINITE = 33
};

struct DecArgs {
  const sif_dec_desc* descs;
  int n;
  uint32_t* table;        // per IF: (2 + max blocks of that stream) rows of TROW_U32
  const uint64_t* tab_off;  // [n+1] start of each stream's table rows (u32 units)
  uint32_t* acc;          // per IF: {crc, flags, count, pad}
  int parse_only;
  int32_t* status;
  const uint32_t* seg_base;    // [n+1] prefix of CRC segments per stream
  const uint64_t* item_base;   // [n+1] prefix of (row, column segment) work items per stream
  int segw;                    // elements per work item (4096)
  const uint32_t* small;       // [n] 1: stream decoded by sif_dec_small (one CTA per stream)
  const uint32_t* small_list;  // the small streams, in batch order
};

constexpr uint64_t SEGD = CRC_PIECE;  // CRC bytes per warp piece

__device__ __forceinline__ uint32_t* dtab(const DecArgs& a, int i) { return a.table + a.tab_off[i]; }
// Stream length as resolved by the parse kernel (table row 1, words 2..3).
__device__ __forceinline__ uint64_t dlen(const uint32_t* tab) {
  return (uint64_t)tab[TROW_U32 + 2] | ((uint64_t)tab[TROW_U32 + 3] << 32);
}

// ------------------------------------------------------------------------------- parse
__device__ __forceinline__ uint32_t rd_u32(const uint8_t* p, uint64_t o) {
  return (uint32_t)p[o] | ((uint32_t)p[o + 1] << 8) | ((uint32_t)p[o + 2] << 16) | ((uint32_t)p[o + 3] << 24);
}

// The stream length comes from the descriptor, or -- for payloads still being produced on
// the device (a pipelined encode -> decode) -- from the encoder's out_len, read here.
// over: the device length exceeds the buffer the stream lives in.
__device__ __forceinline__ uint64_t stream_len(const sif_dec_desc& d, bool& over) {
  over = false;
  if (!d.in_len_dev) return d.in_len;
  const uint64_t l = *d.in_len_dev;
  over = l > d.in_len;
  return over ? 0 : l;
}

// Walk one stream's framing exactly in the order of deserialize (codec.py:320-385) and
// write its block table.  `in` is the stream (device memory, or a shared-memory copy of
// its first len bytes).
// mirror (optional, shared memory): the first mirror_rows table rows are written there too.
__device__ void parse_stream(const DecArgs& a, int i, const uint8_t* in, uint64_t len, bool over,
                             uint32_t* mirror = nullptr, uint32_t mirror_rows = 0) {
  uint32_t* tab = dtab(a, i);
  const uint64_t max_rows = (a.tab_off[i + 1] - a.tab_off[i]) / TROW_U32 - 2;
  uint32_t pre = 0, walk = 0, N = 0, K = 0, mp = 0, mm = 0, mode = 0, qb = 0, nb = 0, crc = 0;
  uint32_t pre_r = R_NONE, walk_r = R_NONE, walk_x = 0;
  if (over) { pre = SIF_ERR_CAPACITY; pre_r = R_LEN_OVER; }  // longer than the buffer it lives in
  else if (len < (uint64_t)(kHeaderBytes + kCrcBytes)) { pre = SIF_ERR_STREAM_FORMAT; pre_r = R_SHORT; }  // codec.py:321
  else if (in[0] != 'S' || in[1] != 'I' || in[2] != 'F' || in[3] != '1') { pre = SIF_ERR_STREAM_FORMAT; pre_r = R_MAGIC; }
  if (!pre) {
    crc = rd_u32(in, len - 4);
    const uint32_t ver = (uint32_t)in[4] | ((uint32_t)in[5] << 8);
    N = rd_u32(in, 6);
    K = rd_u32(in, 10);
    qb = in[22];
    mode = in[27];
    mp = (uint32_t)in[28] | ((uint32_t)in[29] << 8);
    mm = (uint32_t)in[30] | ((uint32_t)in[31] << 8);
    if (ver != 1) { walk = SIF_ERR_STREAM_FORMAT; walk_r = R_VERSION; walk_x = ver; }  // codec.py:331-332
    else if (mode > 1) { walk = SIF_ERR_STREAM_FORMAT; walk_r = R_MODE; walk_x = mode; }  // codec.py:333-334
    else {
      uint64_t pos = kHeaderBytes;
      if (mode == 1) {
        if (len < pos + mp + mm) { walk = SIF_ERR_STREAM_FORMAT; walk_r = R_QVEC; }  // codec.py:340-341
        pos += mp + mm;
      }
      const uint32_t cb = col_bits(K);
      const uint64_t nblk = (uint64_t)mp + mm;
      for (uint64_t b = 0; b < nblk && !walk; ++b) {
        if (len < pos + kBlockMetaBytes + 4ull * ((uint64_t)N + 1)) { walk = SIF_ERR_STREAM_FORMAT; walk_r = R_BLKHDR; break; }
        const uint32_t q = in[pos];
        if (q < 1 || q > (uint32_t)kQMax) { walk = SIF_ERR_CORRUPT_STREAM; walk_r = R_QRANGE; walk_x = q; break; }  // :351-352
        const uint32_t o = rd_u32(in, pos + 1), vmin = rd_u32(in, pos + 5), nnz = rd_u32(in, pos + 9);
        const uint64_t rp = pos + kBlockMetaBytes;
        pos = rp + 4ull * ((uint64_t)N + 1);
        const uint64_t cbytes = ((uint64_t)nnz * cb + 7) / 8, qbytes = ((uint64_t)nnz * q + 7) / 8;
        if (len - kCrcBytes < pos + cbytes + qbytes) { walk = SIF_ERR_STREAM_FORMAT; walk_r = R_BLKPAY; break; }  // :358
        if (b >= max_rows) { walk = SIF_ERR_CAPACITY; walk_r = R_CAPACITY; break; }
        const uint32_t rv[10] = {q, nnz, o, vmin, (uint32_t)rp, (uint32_t)(rp >> 32), (uint32_t)pos,
                                 (uint32_t)(pos >> 32), (uint32_t)(pos + cbytes), (uint32_t)((pos + cbytes) >> 32)};
        uint32_t* row = tab + (2 + b) * TROW_U32;
        for (int k = 0; k < 10; ++k) row[k] = rv[k];
        if (2 + b < mirror_rows)
          for (int k = 0; k < 10; ++k) mirror[(2 + b) * TROW_U32 + k] = rv[k];
        pos += cbytes + qbytes;
      }
      if (!walk && pos != len - kCrcBytes) { walk = SIF_ERR_STREAM_FORMAT; walk_r = R_TRAIL; }  // codec.py:384-385
      nb = (uint32_t)nblk;
    }
  }
  const uint32_t h0[8] = {walk, N, K, mp, mm, mode, qb, nb};
  const uint32_t h1[10] = {pre, crc, (uint32_t)len, (uint32_t)(len >> 32), pre_r, walk_r, walk_x, 0u, 0u,
                           len >= 4 ? rd_u32(in, 0) : 0u};  // [9]: magic bytes for the error message
  for (int k = 0; k < 8; ++k) tab[k] = h0[k];
  for (int k = 0; k < 10; ++k)
    if (k != 7 && k != 8) tab[TROW_U32 + k] = h1[k];  // 7, 8: reason, set by the final pass
  if (mirror_rows >= 2) {
    for (int k = 0; k < 8; ++k) mirror[k] = h0[k];
    for (int k = 0; k < 10; ++k) mirror[TROW_U32 + k] = h1[k];
  }
}

__global__ void sif_parse_kernel(DecArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n || (a.small && a.small[i])) return;  // small streams: sif_dec_small
  const sif_dec_desc d = a.descs[i];
  bool over;
  const uint64_t len = stream_len(d, over);
  parse_stream(a, i, d.in, len, over);
}

// ------------------------------------------------------------------------------- CRC
// One warp per 2 KiB CRC-32 piece of a stream (pieces aligned to the end of [4, len-4)):
// raw piece CRC shifted over the pieces after it (kPieceShift) and XOR-combined into the
// stream's accumulator (GF(2) linearity).
__global__ void __launch_bounds__(DNT, 8) sif_dcrc_kernel(DecArgs a) {
  __shared__ uint32_t t4[1024];
  __shared__ uint32_t stage[DNT / 32][544];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < 1024; k += DNT) t4[k] = (&kCrcTab4[0][0])[k];
  __syncthreads();
  // each warp takes a contiguous range of the pieces (streams walked forward)
  const uint64_t GW = (uint64_t)gridDim.x * (DNT / 32), gw = (uint64_t)blockIdx.x * (DNT / 32) + w;
  const uint64_t total = a.seg_base[a.n];
  const uint64_t p0 = total * gw / GW, p1 = total * (gw + 1) / GW;
  PieceWalk pw;
  pw.init(a.seg_base, a.n);
  for (uint64_t gp = p0; gp < p1; ++gp) {
    const int ifi = pw.at(gp);
    const uint32_t piece = (uint32_t)(gp - pw.b0);
    const uint32_t* tab = dtab(a, ifi);
    if (tab[TROW_U32 + 0]) continue;  // length / magic failure: no CRC
    const sif_dec_desc d = a.descs[ifi];
    // pieces are planned from the buffer capacity; those past the real length exit here
    const uint64_t b0 = 4, b1 = dlen(tab) - 4;
    const uint64_t e1 = (uint64_t)piece * SEGD < b1 - b0 ? b1 - (uint64_t)piece * SEGD : b0;
    const uint64_t e0 = e1 - b0 > SEGD ? e1 - SEGD : b0;
    if (e0 >= e1) continue;
    const uint32_t raw = crc_piece_warp(d.in, e0, e1, t4, stage[w]);
    if (lane == 0 && raw) atomicXor(a.acc + 4ull * ifi + 0, crc_mult(kPieceShift[piece], raw));
  }
}

// Float64 value of the plus-plane entry at (row, col), 0 if none (slow path for elements
// present in both planes).  Plus blocks are 0 .. mp-1; cols are ascending within a row.
__device__ __noinline__ double plus_value(const uint32_t* tab, const uint8_t* in, uint32_t mp, uint32_t r,
                                          uint32_t col, uint32_t cb) {
  double v = 0.0;
  for (uint32_t b = 0; b < mp; ++b) {
    const uint32_t* row = tab + (2ull + b) * TROW_U32;
    const uint32_t q = row[0], nnz = row[1];
    const uint64_t rpo = (uint64_t)row[4] | ((uint64_t)row[5] << 32);
    const uint64_t cbit = 8ull * ((uint64_t)row[6] | ((uint64_t)row[7] << 32));
    const uint64_t qbit = 8ull * ((uint64_t)row[8] | ((uint64_t)row[9] << 32));
    uint32_t lo = min(ld_u32_le(in, rpo + 4ull * r), nnz), hi = min(ld_u32_le(in, rpo + 4ull * (r + 1)), nnz);
    while (lo < hi) {
      const uint32_t m = (lo + hi) >> 1;
      const uint32_t cm = ld_field(in, cbit + (uint64_t)m * cb, cb);
      if (cm == col) {
        const uint32_t code = ld_field(in, qbit + (uint64_t)m * q, q);
        v = __dadd_rn(v, __dadd_rn(__dmul_rn((double)code, (double)__uint_as_float(row[2])),
                                   (double)__uint_as_float(row[3])));
        break;
      }
      if (cm < col) lo = m + 1; else hi = m;
    }
  }
  return v;
}

// ------------------------------------------------------------------------------- scatter
// Corrupt-stream reasons are ranked like the reference's validation order (codec.py:235-251:
// blocks in plane order, inside a block the five checks in order); the IF keeps the first
// one (atomicMax of its complement in acc[3]) so the error message names the same check.
enum : uint32_t { CK_ROWPTR = 0, CK_ROWPTR_NNZ = 1, CK_COL_RANGE = 2, CK_COL_ORDER = 3, CK_OVERLAP = 4 };
__device__ __forceinline__ uint32_t corrupt_key(uint32_t b, uint32_t check) { return b * 8u + check; }

__device__ __forceinline__ void flush_flags(const DecArgs& a, int cur, uint32_t fl, uint32_t ck) {
  fl = __reduce_or_sync(0xFFFFFFFFu, fl);
  ck = __reduce_min_sync(0xFFFFFFFFu, ck);
  if ((threadIdx.x & 31) == 0) {
    if (ck != 0xFFFFFFFFu) {
      fl |= FLAG_CORRUPT;
      atomicMax(a.acc + 4ull * cur + 3, 0xFFFFFFFFu - ck);
    }
    if (fl) atomicOr(a.acc + 4ull * cur + 1, fl);
  }
}

// Work item = (stream, row group, column segment): R = max(1, segw / K) consecutive rows of
// at most segw columns; a warp owns a contiguous range of items.  Lanes hold one (block,
// row) pair each (pairs block-major, plus blocks first, in groups of 32): block metadata
// and the row's entry range, staged in shared memory.  The pairs' entries are unpacked 32
// at a time (cols, codes), validated (codec.py:238-250), dequantized in float64
// (quant.py:67-73) and stored in place: the item's output (contiguous) is zero-filled with
// 16-byte stores first, then each entry's value is written while those lines are still in
// L2, so DRAM sees every output line once.  An element held by one plane is f32(0 +/- v),
// exactly the reference's f64 scatter-add rounded to fp32 (codec.py:257-266); an element
// held by both planes is summed in float64 (plus value recovered from its block).  Within a
// window plus entries are written before minus entries.  Shared memory holds only the
// per-item plane bitmaps (overlap checks), so items are up to 4096 elements.
__global__ void __launch_bounds__(DNT, 3) sif_scatter_kernel(DecArgs a) {
  extern __shared__ __align__(16) uint8_t dsm_raw[];
  __shared__ uint4 pa[DNT / 32][32], pb[DNT / 32][32];
  __shared__ uint2 pc[DNT / 32][32];
  __shared__ uint8_t own[DNT / 32][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t segw = (uint32_t)a.segw;
  const uint32_t bmw = (segw + 31) / 32;
  uint32_t* bm = reinterpret_cast<uint32_t*>(dsm_raw) + (size_t)w * 2 * bmw;
  const uint64_t GW = (uint64_t)gridDim.x * (DNT / 32);
  const uint64_t gw = (uint64_t)blockIdx.x * (DNT / 32) + w;
  const uint64_t nitems = a.item_base[a.n];
  const uint64_t i0 = nitems * gw / GW, i1 = nitems * (gw + 1) / GW;
  int cur = -1;
  uint32_t N = 0, K = 0, mp = 0, nb = 0, nsegr = 1, cb = 1, R = 1;
  uint64_t ib0 = 0, ib1 = 0;
  bool ok = false;
  const uint32_t* tab = nullptr;
  const uint8_t* in = nullptr;
  float* out = nullptr;
  uint32_t fl = 0;
  uint32_t ck = 0xFFFFFFFFu;  // first failing (block, check) of this warp's part of the IF
  for (uint64_t it = i0; it < i1; ++it) {
    if (cur < 0 || it >= ib1) {
      if (cur >= 0) flush_flags(a, cur, fl, ck);
      fl = 0;
      ck = 0xFFFFFFFFu;
      int lo = cur < 0 ? 0 : cur, hi = a.n - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (a.item_base[mid] <= it) lo = mid; else hi = mid - 1;
      }
      cur = lo;
      ib0 = a.item_base[cur];
      ib1 = a.item_base[cur + 1];
      const sif_dec_desc d = a.descs[cur];
      tab = dtab(a, cur);
      const uint32_t walk = tab[0], pre = tab[TROW_U32 + 0];
      N = tab[1]; K = tab[2]; mp = tab[3]; nb = tab[7];
      ok = !pre && !walk && N == d.rows && K == d.cols && !a.parse_only;
      in = d.in;
      out = d.out;
      nsegr = (d.cols + segw - 1) / segw;
      R = d.cols <= segw ? segw / d.cols : 1u;
      cb = col_bits(K);
    }
    if (!ok) continue;
    const uint64_t li = it - ib0;
    uint32_t rg, sg;
    if (nsegr == 1) { rg = (uint32_t)li; sg = 0; }
    else { rg = (uint32_t)(li / nsegr); sg = (uint32_t)(li - (uint64_t)rg * nsegr); }
    const uint32_t r0 = rg * R, nr = min(R, N - r0);
    const uint32_t c0 = sg * segw, c1 = min(K, c0 + segw), W = c1 - c0;
    const uint32_t span = nr * W;  // item elements (rows are contiguous when nsegr == 1)
    for (uint32_t k = lane; k < 2 * bmw; k += 32) bm[k] = 0;
    // the item's output is zero-filled first (coalesced), then every entry's value is
    // stored in place while the lines are still in L2 (row r0 + ri, column col)
    // (the item is contiguous: whole rows when W == K, else a single row segment)
    float* dst = out + (uint64_t)r0 * K + c0;
    if ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0 && (span & 3u) == 0) {
      for (uint32_t k = 4 * lane; k < span; k += 128) *reinterpret_cast<float4*>(dst + k) = make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      for (uint32_t k = lane; k < span; k += 32) dst[k] = 0.f;
    }
    __syncwarp();
    uint32_t nf0 = 0;  // a plus-plane value rounded to a non-finite fp32 (re-checked at the store)
    const uint32_t np = nb * nr;       // (block, row) pairs, block-major
    for (uint32_t g0 = 0; g0 < np; g0 += 32) {
      const uint32_t g1 = min(np, g0 + 32u);
      const uint32_t pi = g0 + lane;
      uint32_t cnt = 0;
      if (pi < g1) {
        const uint32_t b = pi / nr;
        const uint32_t ri = pi - b * nr;
        const uint32_t r = r0 + ri;
        const uint4* row4 = reinterpret_cast<const uint4*>(tab + (2ull + b) * TROW_U32);
        const uint4 m0v = row4[0], m1v = row4[1];
        const uint32_t q = m0v.x, nnz = m0v.y;
        const uint64_t rpo = (uint64_t)m1v.x | ((uint64_t)m1v.y << 32);
        const uint64_t cbit = 8ull * ((uint64_t)m1v.z | ((uint64_t)m1v.w << 32));
        const uint2 m2v = *reinterpret_cast<const uint2*>(tab + (2ull + b) * TROW_U32 + 8);
        const uint64_t qbit = 8ull * ((uint64_t)m2v.x | ((uint64_t)m2v.y << 32));
        const uint32_t p0 = ld_u32_le(in, rpo + 4ull * r), p1 = ld_u32_le(in, rpo + 4ull * (r + 1));
        if (sg == 0) {
          if (r == 0 && p0 != 0) ck = min(ck, corrupt_key(b, CK_ROWPTR));  // codec.py:238-239
          if (p1 < p0 || (r + 1 == N && p1 != nnz)) ck = min(ck, corrupt_key(b, CK_ROWPTR_NNZ));  // :240-241
        }
        uint32_t lo = min(p0, nnz), hi = max(lo, min(p1, nnz));
        const uint32_t rs0 = lo;
        if (nsegr > 1) {
          // entries of this column segment: lower bounds of c0 and c1 among the row's cols
          auto lb = [&](uint32_t cv) {
            uint32_t a0 = lo, a1 = hi;
            while (a0 < a1) {
              const uint32_t m = (a0 + a1) >> 1;
              if (ld_field(in, cbit + (uint64_t)m * cb, cb) < cv) a0 = m + 1; else a1 = m;
            }
            return a0;
          };
          const uint32_t l0 = sg == 0 ? lo : lb(c0);
          const uint32_t l1 = sg + 1 == nsegr ? hi : lb(c1);
          lo = l0;
          hi = max(l0, l1);
        }
        cnt = hi - lo;
        // pair parameters in shared memory (entry base stored as lo - exclusive prefix)
        pa[w][lane] = make_uint4((uint32_t)cbit, (uint32_t)(cbit >> 32), (uint32_t)qbit, (uint32_t)(qbit >> 32));
        pb[w][lane] = make_uint4(lo, q, m0v.z, m0v.w);
        pc[w][lane] = make_uint2(rs0, ri | (b << 12) | (b >= mp ? 0x80000000u : 0u));  // ri < R <= segw = 4096
      }
      const uint32_t inc = warp_incl_scan_u32(cnt);
      const uint32_t M = __shfl_sync(0xFFFFFFFFu, inc, 31);
      const uint32_t exc = inc - cnt;
      if (pi < g1) pb[w][lane].x -= exc;
      uint32_t lastcol = 0, lastjl = 0xFFFFFFFFu;
      // window m0: owner pair of entry m0 + lane, its parameters and its col / code fields.
      // The fields of window m0 + 32 are fetched while window m0 is processed (two
      // memory round trips in flight per warp).
      struct Win {
        uint32_t jl, e, col, code;  // the rest of the pair's parameters is re-read from smem
      };
      auto prep = [&](uint32_t m0, Win& x) {
        const uint32_t m = m0 + lane;
        // owner of entry m: the last pair (with entries) starting at or before m in this
        // window; window position 0 is owned by the pair covering m0
        const uint32_t st0 = max(exc, m0);
        const bool starts = cnt != 0 && st0 < inc && st0 < m0 + 32u;
        if (starts) own[w][st0 - m0] = (uint8_t)lane;
        const uint32_t smask = __reduce_or_sync(0xFFFFFFFFu, starts ? 1u << (st0 - m0) : 0u);
        __syncwarp();
        const uint32_t src = 31u - __clz(smask & (0xFFFFFFFFu >> (31 - lane)));
        x.jl = own[w][src];
        const uint4 A = pa[w][x.jl];
        const uint2 Bxy = *reinterpret_cast<const uint2*>(&pb[w][x.jl]);  // entry base, q
        const uint64_t cbj = (uint64_t)A.x | ((uint64_t)A.y << 32);
        x.e = Bxy.x + m;
        const uint64_t qbj = (uint64_t)A.z | ((uint64_t)A.w << 32);
        x.col = 0;
        x.code = 0;
        if (m < M) {
          // byte fields (8-bit cols when K <= 256, 8-bit codes) are single byte loads
          x.col = cb == 8 ? (uint32_t)__ldg(in + (cbj >> 3) + x.e) : ld_field(in, cbj + (uint64_t)x.e * cb, cb);
          x.code = Bxy.y == 8 ? (uint32_t)__ldg(in + (qbj >> 3) + x.e) : ld_field(in, qbj + (uint64_t)x.e * Bxy.y, Bxy.y);
        }
      };
      Win cw;
      if (M > 0) prep(0, cw);
      for (uint32_t m0 = 0; m0 < M; m0 += 32) {
        const uint32_t m = m0 + lane;
        Win nw;
        const bool more = m0 + 32 < M;
        __syncwarp();  // every lane has read own[] for window m0
        if (more) prep(m0 + 32, nw);
        const uint32_t jl = cw.jl, e = cw.e, col = cw.col, code = cw.code;
        const uint2 C = pc[w][jl];
        const uint32_t rij = C.y & 0xFFFu, bj = (C.y >> 12) & 0x7FFFFu;
        const bool minus = (C.y >> 31) != 0;
        // the previous entry e-1 of the same pair sits in the previous lane of this window
        // (lane 0: the last lane of the previous window)
        uint32_t colp = __shfl_up_sync(0xFFFFFFFFu, col, 1);
        uint32_t jlp = __shfl_up_sync(0xFFFFFFFFu, jl, 1);
        if (lane == 0) { colp = lastcol; jlp = lastjl; }
        lastcol = __shfl_sync(0xFFFFFFFFu, col, 31);
        lastjl = __shfl_sync(0xFFFFFFFFu, jl, 31);
        bool wr = false;
        uint32_t pos = 0;
        double v = 0.0;
        if (m < M) {
          if (col >= K) ck = min(ck, corrupt_key(bj, CK_COL_RANGE));  // codec.py:242-243
          else {
            // strictly increasing within the row (codec.py:244-247)
            if (e > C.x) {
              const uint64_t cbj = (uint64_t)pa[w][jl].x | ((uint64_t)pa[w][jl].y << 32);
              const uint32_t prev = jlp == jl ? colp : ld_field(in, cbj + (uint64_t)(e - 1) * cb, cb);
              if (prev >= col) ck = min(ck, corrupt_key(bj, CK_COL_ORDER));
            }
            if (col >= c0 && col < c1) {
              wr = true;
              pos = rij * W + (col - c0);
              const uint32_t old = atomicOr(bm + (minus ? bmw : 0u) + (pos >> 5), 1u << (pos & 31));
              if (old & (1u << (pos & 31))) {  // codec.py:248-250 (corrupt: the first value stays)
                ck = min(ck, corrupt_key(bj, CK_OVERLAP));
                wr = false;
              }
              const uint2 ov = *reinterpret_cast<const uint2*>(&pb[w][jl].z);  // o, v_min
              v = __dadd_rn(__dmul_rn((double)code, (double)__uint_as_float(ov.x)), (double)__uint_as_float(ov.y));
              if (wr && !minus) {
                const float f = __double2float_rn(v);  // f32(0 + v)
                dst[pos] = f;
                nf0 |= (__float_as_uint(f) & 0x7F800000u) == 0x7F800000u ? 1u : 0u;
              }
            }
          }
        }
        __syncwarp();  // plus entries of this window land before the minus entries read them
        if (wr && minus) {
          float f;
          if ((bm[pos >> 5] >> (pos & 31)) & 1u) {
            // both planes hold this element: the reference sums them in float64
            // (codec.py:257-266); recover the plus value from its plus block entry
            const double pv = plus_value(tab, in, mp, r0 + rij, col, cb);
            f = __double2float_rn(__dsub_rn(pv, v));
          } else {
            f = __double2float_rn(-v);  // f32(0 - v)
          }
          dst[pos] = f;
          if ((__float_as_uint(f) & 0x7F800000u) == 0x7F800000u) fl |= FLAG_NONFINITE;
        }
        __syncwarp();
        if (more) cw = nw;
      }
    }
    // a non-finite plus value may have been summed with a minus entry since: re-check the
    // item's final values (rare)
    uint32_t bad = 0;
    if (__any_sync(0xFFFFFFFFu, nf0 != 0)) {
      __syncwarp();
      for (uint32_t k = lane; k < span; k += 32) bad |= (__float_as_uint(dst[k]) & 0x7F800000u) == 0x7F800000u ? 1u : 0u;
    }
    if (bad) fl |= FLAG_NONFINITE;
    __syncwarp();
  }
  if (cur >= 0) flush_flags(a, cur, fl, ck);
}

// ------------------------------------------------------------------------------- small streams
// sif_dec_small: one CTA per stream whose dense output fits in shared memory (rows * cols
// <= SMALL_T; a decode-step token 1 x 4096, or any small IF) -- the whole decode of the
// stream in one launch for the batch.  The stream (up to SMALL_CAP bytes) is copied into
// shared memory once; the framing walk (parse_stream), CRC, row_ptr / cols validation
// (codec.py:235-251), unpack, float64 dequantize (quant.py:67-73) and the fp32 dense
// buffer (codec.py:257-266) all work from shared memory, and the output is written with
// one coalesced pass.  Same block table, reason codes and error precedence as the
// four-kernel path (sif_dfinal_kernel).
constexpr int DSN = 128;             // threads per small-stream CTA
constexpr uint32_t SMALL_T = 4096;   // max dense elements of a small stream
constexpr uint32_t SMALL_CAP = 4096; // stream bytes staged in shared memory
constexpr uint32_t SMALL_ROWS = 34;  // table rows mirrored in shared memory (2 + 32 blocks)

// Generic-address versions of ld_u32_le / ld_field (the shared-memory copy or the stream
// itself; base 4-byte aligned).
__device__ __forceinline__ uint32_t gen_u32_le(const uint8_t* base, uint64_t off) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(base);
  const uint64_t wi = off >> 2;
  const uint32_t sh = 8u * (uint32_t)(off & 3u);
  const uint32_t lo = w[wi];
  return sh ? __funnelshift_r(lo, w[wi + 1], sh) : lo;
}
__device__ __forceinline__ uint32_t gen_field(const uint8_t* base, uint64_t bit, uint32_t wd) {
  const uint32_t* p = reinterpret_cast<const uint32_t*>(base);
  const uint64_t wi = bit >> 5;
  const uint32_t sh = (uint32_t)(bit & 31u);
  uint64_t hi = (uint64_t)bswap32(p[wi]) << 32;
  if (sh + wd > 32u) hi |= bswap32(p[wi + 1]);
  return (uint32_t)((hi << sh) >> (64u - wd));
}

struct SmallSh {
  float buf[SMALL_T];                 // the dense output (first: the CRC staging area)
  uint32_t bm[2][SMALL_T / 32];       // elements written by the plus / minus plane
  uint32_t t4[1024];                  // CRC slice tables
  uint32_t cp[SMALL_CAP / 4 + 4];     // the stream, zero padded
  uint32_t tab[SMALL_ROWS * TROW_U32]; // the first table rows (header + blocks)
  uint32_t pre[SMALL_ROWS];            // nnz prefix over the blocks
  uint32_t ovl;                        // a plane overlap seen in the flattened pass
  uint32_t red[DSN / 32 + 1];
  uint32_t ck, fl, crcok;
  uint64_t bar;                        // mbarrier of the bulk stream copy
};

__global__ void __launch_bounds__(DSN, 7) sif_dec_small(DecArgs a) {
  __shared__ __align__(16) SmallSh sh;
  static_assert(DSN * 16 <= SMALL_T, "CRC staging must fit the dense buffer");
  const int tid = threadIdx.x, lane = tid & 31;
  const int i = (int)a.small_list[blockIdx.x];
  const sif_dec_desc d = a.descs[i];
  bool over;
  const uint64_t len = stream_len(d, over);
  const bool staged = len <= SMALL_CAP;
  // stage the stream: a 16-byte aligned stream's whole 16-byte part by one bulk-async copy
  // (cp.async.bulk, completing on an mbarrier), the rest (tail, zero padding) by plain loads
  const bool bulk = staged && (reinterpret_cast<uintptr_t>(d.in) & 15u) == 0 && len >= 16;
  const uint32_t nb16 = bulk ? (uint32_t)(len & ~15ull) : 0u;
  if (bulk && tid == 0) {
    mbar_init(&sh.bar, 1);
    bulk_copy_g2s(sh.cp, d.in, nb16, &sh.bar);
  }
  if (staged) {
    const uint32_t* gw = reinterpret_cast<const uint32_t*>(d.in);
    const uint32_t nfull = (uint32_t)(len / 4), nw = (uint32_t)((len + 3) / 4);
    for (uint32_t k = nb16 / 4 + tid; k < nw + 4; k += DSN) {
      uint32_t v = 0;
      if (k < nfull) v = __ldg(gw + k);
      else if (k < nw)  // the partial last word: byte loads (nothing past the stream is read)
        for (uint32_t b = 0; 4 * k + b < len; ++b) v |= (uint32_t)__ldg(d.in + 4 * k + b) << (8 * b);
      sh.cp[k] = v;
    }
  }
  for (int k = tid; k < 1024; k += DSN) sh.t4[k] = (&kCrcTab4[0][0])[k];
  if (tid == 0) { sh.ck = 0xFFFFFFFFu; sh.fl = 0; }
  __syncthreads();  // (orders the barrier's init before the other threads wait on it)
  if (bulk) mbar_wait_parity(&sh.bar, 0);
  const uint8_t* src = staged ? reinterpret_cast<const uint8_t*>(sh.cp) : d.in;
  if (tid == 0) parse_stream(a, i, src, len, over, sh.tab, SMALL_ROWS);
  __syncthreads();  // the table rows written by thread 0 are visible to the CTA
  uint32_t* gtab = dtab(a, i);
  const uint32_t pre = sh.tab[TROW_U32 + 0];
  uint32_t crc_raw = 0;
  if (!pre) {
    uint32_t* cst = reinterpret_cast<uint32_t*>(sh.buf);
    crc_raw = staged ? crc_cta_pieces<DSN, true>(src, 4, len - 4, sh.t4, sh.red, cst)
                     : crc_cta_pieces<DSN>(d.in, 4, len - 4, sh.t4, sh.red, cst);
  }
  if (tid == 0) sh.crcok = (!pre && crc_finish(crc_raw, len - 8) == sh.tab[TROW_U32 + 1]) ? 1u : 0u;
  __syncthreads();
  const bool crc_ok = sh.crcok != 0;
  const uint32_t walk = sh.tab[0], N = sh.tab[1], K = sh.tab[2], mp = sh.tab[3], nb = sh.tab[7];
  // block rows: shared-memory mirror when they all fit, else the global table
  const uint32_t* tab = nb + 2 <= SMALL_ROWS ? sh.tab : gtab;
  const bool shape_ok = a.parse_only || (N == d.rows && K == d.cols);
  const bool ok = crc_ok && !walk && !a.parse_only && N == d.rows && K == d.cols;
  uint32_t ck = 0xFFFFFFFFu, fl = 0, nfp = 0;
  if (ok) {
    const uint32_t T = N * K, cb = col_bits(K);
    for (uint32_t k = tid; k < T; k += DSN) sh.buf[k] = 0.f;
    for (uint32_t k = tid; k < 2 * SMALL_T / 32; k += DSN) (&sh.bm[0][0])[k] = 0u;
    __syncthreads();
    // entry m of block b: row (codec.py:238-241 ranges), col checks (codec.py:242-247),
    // plane overlap (codec.py:248-250), float64 value (quant.py:67-73, codec.py:257-266).
    // exact == false: an overlap only raises the plane's redo flag (the entries of a plane
    // run in parallel, so which block saw the collision first is not the reference's order)
    auto entry = [&](uint32_t b, uint32_t m, bool exact) {
      const uint32_t* row = tab + (2ull + b) * TROW_U32;
      const uint32_t q = row[0];
      const uint64_t rpo = (uint64_t)row[4] | ((uint64_t)row[5] << 32);
      const uint64_t cbit = 8ull * ((uint64_t)row[6] | ((uint64_t)row[7] << 32));
      const uint32_t minus = b >= mp ? 1u : 0u;
      // the entry's row: the last r < N with row_ptr[r] <= m
      uint32_t lo = 0, hi = N - 1;
      while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (gen_u32_le(src, rpo + 4ull * mid) <= m) lo = mid; else hi = mid - 1;
      }
      const uint32_t r = lo;
      const uint32_t col = gen_field(src, cbit + (uint64_t)m * cb, cb);
      if (col >= K) { ck = min(ck, corrupt_key(b, CK_COL_RANGE)); return; }  // codec.py:242-243
      if (m > gen_u32_le(src, rpo + 4ull * r) && gen_field(src, cbit + (uint64_t)(m - 1) * cb, cb) >= col)
        ck = min(ck, corrupt_key(b, CK_COL_ORDER));  // codec.py:244-247
      const uint32_t pos = r * K + col, bit = 1u << (pos & 31u);
      if (atomicOr(&sh.bm[minus][pos >> 5], bit) & bit) {  // corrupt: the first value stays
        if (exact) ck = min(ck, corrupt_key(b, CK_OVERLAP));
        else sh.ovl = 1;
        return;
      }
      const uint64_t qbit = 8ull * ((uint64_t)row[8] | ((uint64_t)row[9] << 32));
      const double o = (double)__uint_as_float(row[2]), vmin = (double)__uint_as_float(row[3]);
      const uint32_t code = gen_field(src, qbit + (uint64_t)m * q, q);
      const double v = __dadd_rn(__dmul_rn((double)code, o), vmin);
      float f;
      if (!minus) f = __double2float_rn(v);  // f32(0 + v)
      else if (sh.bm[0][pos >> 5] & bit)  // both planes: summed in float64 (codec.py:257-266)
        f = __double2float_rn(__dsub_rn(plus_value(gtab, d.in, mp, r, col, cb), v));
      else f = __double2float_rn(-v);  // f32(0 - v)
      sh.buf[pos] = f;
      // a minus write is final; a non-finite plus value may still be summed with a minus
      // entry, so it only triggers the full scan below
      if ((__float_as_uint(f) & 0x7F800000u) == 0x7F800000u) {
        if (minus) fl = FLAG_NONFINITE;
        else nfp = 1;
      }
    };
    // row_ptr checks of every block (codec.py:238-241)
    for (uint32_t k = tid; k < nb * N; k += DSN) {
      const uint32_t b = k / N, r = k - b * N;
      const uint32_t* row = tab + (2ull + b) * TROW_U32;
      const uint64_t rpo = (uint64_t)row[4] | ((uint64_t)row[5] << 32);
      const uint32_t p0 = gen_u32_le(src, rpo + 4ull * r), p1 = gen_u32_le(src, rpo + 4ull * (r + 1));
      if (r == 0 && p0 != 0) ck = min(ck, corrupt_key(b, CK_ROWPTR));
      if (p1 < p0 || (r + 1 == N && p1 != row[1])) ck = min(ck, corrupt_key(b, CK_ROWPTR_NNZ));
    }
    // block-ordered pass over the blocks [b0, b1): one barrier per block, overlaps charged to
    // the later block exactly like the reference's `seen` mask
    auto ordered = [&](uint32_t b0, uint32_t b1) {
      for (uint32_t b = b0; b < b1; ++b) {
        const uint32_t nnz = tab[(2ull + b) * TROW_U32 + 1];
        for (uint32_t m = tid; m < nnz; m += DSN) entry(b, m, true);
        __syncthreads();
      }
    };
    if (nb + 2 <= SMALL_ROWS) {
      // the table rows are in shared memory: each plane's entries in one flattened pass
      // (entry i -> block by the nnz prefix); a plane with an overlap (corrupt) is redone
      // in block order for the reference's error
      if (tid == 0) {
        uint32_t acc = 0;
        for (uint32_t b = 0; b < nb; ++b) { sh.pre[b] = acc; acc += tab[(2ull + b) * TROW_U32 + 1]; }
        sh.pre[nb] = acc;
        sh.ovl = 0;
      }
      __syncthreads();
      for (uint32_t pl = 0; pl < 2; ++pl) {
        const uint32_t b0 = pl ? mp : 0u, b1 = pl ? nb : mp;
        if (b0 >= b1) continue;
        const uint32_t i0 = sh.pre[b0], i1 = sh.pre[b1];
        for (uint32_t i = i0 + tid; i < i1; i += DSN) {
          uint32_t b = b0;
          while (b + 1 < b1 && sh.pre[b + 1] <= i) ++b;
          entry(b, i - sh.pre[b], false);
        }
        __syncthreads();
        const bool redo = sh.ovl != 0;
        __syncthreads();  // every thread has read the flag before the next plane may set it
        if (redo) {
          if (tid == 0) sh.ovl = 0;
          for (uint32_t k = tid; k < SMALL_T / 32; k += DSN) sh.bm[pl][k] = 0u;
          __syncthreads();
          ordered(b0, b1);
        }
      }
    } else {
      ordered(0, nb);
    }
    if (__syncthreads_or(nfp))  // non-finite outputs (tensor.py:35-36)
      for (uint32_t k = tid; k < T; k += DSN)
        if ((__float_as_uint(sh.buf[k]) & 0x7F800000u) == 0x7F800000u) fl = FLAG_NONFINITE;
    float* dst = d.out;
    if ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0 && (T & 3u) == 0) {
      for (uint32_t k = 4 * tid; k < T; k += 4 * DSN)
        __stcs(reinterpret_cast<float4*>(dst + k), *reinterpret_cast<const float4*>(sh.buf + k));
    } else {
      for (uint32_t k = tid; k < T; k += DSN) __stcs(dst + k, sh.buf[k]);
    }
  }
  ck = __reduce_min_sync(0xFFFFFFFFu, ck);
  fl = __reduce_or_sync(0xFFFFFFFFu, fl);
  if (lane == 0) {
    if (ck != 0xFFFFFFFFu) atomicMin(&sh.ck, ck);
    if (fl) atomicOr(&sh.fl, fl);
  }
  __syncthreads();
  if (tid == 0) {  // the reference's error precedence (as sif_dfinal_kernel)
    int st = SIF_OK;
    uint32_t r = R_NONE, x = 0;
    if (pre) { st = (int)pre; r = sh.tab[TROW_U32 + 4]; }
    else if (!crc_ok) { st = SIF_ERR_STREAM_FORMAT; r = R_CRC; }  // codec.py:325-327
    else if (walk) { st = (int)walk; r = sh.tab[TROW_U32 + 5]; x = sh.tab[TROW_U32 + 6]; }
    else if (!shape_ok) { st = SIF_ERR_CAPACITY; r = R_SHAPE_MISMATCH; }
    else if (!a.parse_only) {
      if (sh.ck != 0xFFFFFFFFu) { st = SIF_ERR_CORRUPT_STREAM; r = R_CORRUPT + (sh.ck & 7u); x = sh.ck >> 3; }
      else if (N < 1 || K < 1) { st = SIF_ERR_SHAPE; r = R_SHAPE; }
      else if (sh.fl & FLAG_NONFINITE) { st = SIF_ERR_NONFINITE; r = R_NONFINITE; }
    }
    a.status[i] = st;
    gtab[TROW_U32 + 7] = r;
    gtab[TROW_U32 + 8] = x;
  }
}

// Rebind stream i of an uploaded plan (sif_dec_set_input): buffers and device length.
__global__ void set_dec_input_kernel(sif_dec_desc* d, const uint8_t* in, uint64_t* len_slot, uint64_t len, float* out) {
  d->in = in;
  d->out = out;
  *len_slot = len;
  d->in_len_dev = len_slot;
}

// ------------------------------------------------------------------------------- finalize
// One thread per stream: the reference's error precedence (codec.py:320-385, :235-252,
// tensor.py:27-36) from framing, CRC and validation flags; resets the accumulators.
__global__ void sif_dfinal_kernel(DecArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n || (a.small && a.small[i])) return;
  uint32_t* tab = dtab(a, i);
  const sif_dec_desc d = a.descs[i];
  uint32_t* acc = a.acc + 4ull * i;
  const uint32_t walk = tab[0], N = tab[1], K = tab[2], pre = tab[TROW_U32 + 0];
  const uint32_t crc_raw = acc[0], flags = acc[1], ckey = 0xFFFFFFFFu - acc[3];
  const bool shape_ok = a.parse_only || (N == d.rows && K == d.cols);
  int st = SIF_OK;
  uint32_t r = R_NONE, x = 0;
  if (pre) { st = (int)pre; r = tab[TROW_U32 + 4]; }
  else if (crc_finish(crc_raw, dlen(tab) - 8) != tab[TROW_U32 + 1]) { st = SIF_ERR_STREAM_FORMAT; r = R_CRC; }  // :325-327
  else if (walk) { st = (int)walk; r = tab[TROW_U32 + 5]; x = tab[TROW_U32 + 6]; }
  else if (!shape_ok) { st = SIF_ERR_CAPACITY; r = R_SHAPE_MISMATCH; }
  else if (!a.parse_only) {
    if (flags & FLAG_CORRUPT) { st = SIF_ERR_CORRUPT_STREAM; r = R_CORRUPT + (ckey & 7u); x = ckey >> 3; }
    else if (N < 1 || K < 1) { st = SIF_ERR_SHAPE; r = R_SHAPE; }
    else if (flags & FLAG_NONFINITE) { st = SIF_ERR_NONFINITE; r = R_NONFINITE; }
  }
  a.status[i] = st;
  tab[TROW_U32 + 7] = r;
  tab[TROW_U32 + 8] = x;
  acc[0] = 0; acc[1] = 0; acc[2] = 0; acc[3] = 0;
}

}  // namespace sif
