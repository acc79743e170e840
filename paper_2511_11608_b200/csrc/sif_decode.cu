// sif_decode.cu -- B200 (sm_100a) decoder for the SLICER .sif wire format.
//
// Four launches per batch:
//   sif_parse_kernel   one thread per stream walks the header/block framing exactly in the
//                      order of deserialize (codec.py:320-385) and writes a block table.
//   sif_dcrc_kernel    one CTA per 64 KiB CRC-32 segment of a stream (GF(2)-combined).
//   sif_scatter_kernel one warp per (row, column segment): row_ptr/cols validation
//                      (codec.py:235-251), fused unpack + float64 dequantize
//                      (quant.py:67-73) + scatter into a float64 shared-memory row buffer,
//                      rounded to fp32 (codec.py:266) and written once with 16-byte stores.
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
  int segw;                    // columns per work item (<= 1024, multiple of 4)
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

__global__ void sif_parse_kernel(DecArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const sif_dec_desc d = a.descs[i];
  uint32_t* tab = dtab(a, i);
  const uint8_t* in = d.in;
  // the stream length comes from the descriptor, or -- for payloads still being produced on
  // the device (a pipelined encode -> decode) -- from the encoder's out_len, read here
  uint64_t len = d.in_len;
  bool over = false;
  if (d.in_len_dev) {
    const uint64_t l = *d.in_len_dev;
    over = l > d.in_len;
    len = over ? 0 : l;
  }
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
        uint32_t* row = tab + (2 + b) * TROW_U32;
        row[0] = q; row[1] = nnz; row[2] = o; row[3] = vmin;
        row[4] = (uint32_t)rp; row[5] = (uint32_t)(rp >> 32);
        row[6] = (uint32_t)pos; row[7] = (uint32_t)(pos >> 32);
        row[8] = (uint32_t)(pos + cbytes); row[9] = (uint32_t)((pos + cbytes) >> 32);
        pos += cbytes + qbytes;
      }
      if (!walk && pos != len - kCrcBytes) { walk = SIF_ERR_STREAM_FORMAT; walk_r = R_TRAIL; }  // codec.py:384-385
      nb = (uint32_t)nblk;
    }
  }
  tab[0] = walk; tab[1] = N; tab[2] = K; tab[3] = mp; tab[4] = mm; tab[5] = mode; tab[6] = qb; tab[7] = nb;
  tab[TROW_U32 + 0] = pre;
  tab[TROW_U32 + 1] = crc;
  tab[TROW_U32 + 2] = (uint32_t)len;
  tab[TROW_U32 + 3] = (uint32_t)(len >> 32);
  tab[TROW_U32 + 4] = pre_r;
  tab[TROW_U32 + 5] = walk_r;
  tab[TROW_U32 + 6] = walk_x;
  tab[TROW_U32 + 9] = len >= 4 ? rd_u32(in, 0) : 0u;  // magic bytes for the error message
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
  const uint64_t GW = (uint64_t)gridDim.x * (DNT / 32);
  const uint64_t total = a.seg_base[a.n];
  for (uint64_t gp = (uint64_t)blockIdx.x * (DNT / 32) + w; gp < total; gp += GW) {
    int lo = 0, hi = a.n - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (a.seg_base[mid] <= gp) lo = mid; else hi = mid - 1;
    }
    const int ifi = lo;
    const uint32_t piece = (uint32_t)(gp - a.seg_base[lo]);
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
// (quant.py:67-73) into a per-warp fp32 buffer: an element held by one plane is
// f32(0 +/- v), exactly the reference's f64 scatter-add rounded to fp32 (codec.py:257-266);
// an element held by both planes is summed in float64 (plus value recovered from its
// block).  Within a window plus entries are written before minus entries.  The buffer is
// stored with 16-byte streaming stores and re-zeroed in the same pass.
__global__ void __launch_bounds__(DNT, 3) sif_scatter_kernel(DecArgs a) {
  extern __shared__ __align__(16) uint8_t dsm_raw[];
  __shared__ uint4 pa[DNT / 32][32], pb[DNT / 32][32];
  __shared__ uint2 pc[DNT / 32][32];
  __shared__ uint8_t own[DNT / 32][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t segw = (uint32_t)a.segw;
  const uint32_t bmw = (segw + 31) / 32;
  float* buf = reinterpret_cast<float*>(dsm_raw) + (size_t)w * segw;
  uint32_t* bm = reinterpret_cast<uint32_t*>(reinterpret_cast<float*>(dsm_raw) + (size_t)(DNT / 32) * segw) +
                 (size_t)w * 2 * bmw;
  for (uint32_t k = 4 * lane; k < segw; k += 128) *reinterpret_cast<float4*>(buf + k) = make_float4(0.f, 0.f, 0.f, 0.f);
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
    const uint32_t span = nr * W;  // buffer elements (rows are contiguous when nsegr == 1)
    for (uint32_t k = lane; k < 2 * bmw; k += 32) bm[k] = 0;
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
        pc[w][lane] = make_uint2(rs0, ri | (b << 11) | (b >= mp ? 0x80000000u : 0u));  // ri < segw <= 2047
      }
      const uint32_t inc = warp_incl_scan_u32(cnt);
      const uint32_t M = __shfl_sync(0xFFFFFFFFu, inc, 31);
      const uint32_t exc = inc - cnt;
      if (pi < g1) pb[w][lane].x -= exc;
      uint32_t lastcol = 0, lastjl = 0xFFFFFFFFu;
      for (uint32_t m0 = 0; m0 < M; m0 += 32) {
        const uint32_t m = m0 + lane;
        // owner of entry m: the last pair (with entries) starting at or before m in this
        // window; window position 0 is owned by the pair covering m0
        const uint32_t st0 = max(exc, m0);
        const bool starts = cnt != 0 && st0 < inc && st0 < m0 + 32u;
        if (starts) own[w][st0 - m0] = (uint8_t)lane;
        const uint32_t smask = __reduce_or_sync(0xFFFFFFFFu, starts ? 1u << (st0 - m0) : 0u);
        __syncwarp();
        const uint32_t src = 31u - __clz(smask & (0xFFFFFFFFu >> (31 - lane)));
        const uint32_t jl = own[w][src];
        const uint4 A = pa[w][jl];
        const uint4 B = pb[w][jl];
        const uint2 C = pc[w][jl];
        const uint64_t cbj = (uint64_t)A.x | ((uint64_t)A.y << 32);
        const uint32_t e = B.x + m;
        const uint32_t rij = C.y & 0x7FFu, bj = (C.y >> 11) & 0xFFFFFu;
        const bool minus = (C.y >> 31) != 0;
        // col and code fields are fetched together (one memory round trip per window)
        const uint64_t qbj = (uint64_t)A.z | ((uint64_t)A.w << 32);
        uint32_t col = 0, code = 0;
        if (m < M) {
          // IFs with 8-bit cols (K <= 256): byte fields are single byte loads
          if (cb == 8) {
            col = (uint32_t)__ldg(in + (cbj >> 3) + e);
            code = B.y == 8 ? (uint32_t)__ldg(in + (qbj >> 3) + e) : ld_field(in, qbj + (uint64_t)e * B.y, B.y);
          } else {
            col = ld_field(in, cbj + (uint64_t)e * cb, cb);
            code = ld_field(in, qbj + (uint64_t)e * B.y, B.y);
          }
        }
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
              const uint32_t prev = jlp == jl ? colp : ld_field(in, cbj + (uint64_t)(e - 1) * cb, cb);
              if (prev >= col) ck = min(ck, corrupt_key(bj, CK_COL_ORDER));
            }
            if (col >= c0 && col < c1) {
              wr = true;
              pos = rij * W + (col - c0);
              const uint32_t old = atomicOr(bm + (minus ? bmw : 0u) + (pos >> 5), 1u << (pos & 31));
              if (old & (1u << (pos & 31))) ck = min(ck, corrupt_key(bj, CK_OVERLAP));  // codec.py:248-250
              v = __dadd_rn(__dmul_rn((double)code, (double)__uint_as_float(B.z)), (double)__uint_as_float(B.w));
              if (!minus) {
                const float f = __double2float_rn(v);  // f32(0 + v)
                buf[pos] = f;
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
          buf[pos] = f;
          if ((__float_as_uint(f) & 0x7F800000u) == 0x7F800000u) fl |= FLAG_NONFINITE;
        }
        __syncwarp();
      }
    }
    // store (nr full rows, or one row segment) and re-zero the buffer
    const bool chk = __any_sync(0xFFFFFFFFu, nf0 != 0);
    float* dst = out + (uint64_t)r0 * K + c0;
    uint32_t bad = 0;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    if ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0 && (span & 3u) == 0) {
      for (uint32_t k = 4 * lane; k < span; k += 128) {
        const float4 f = *reinterpret_cast<const float4*>(buf + k);
        *reinterpret_cast<float4*>(buf + k) = z4;
        if (chk)
          bad |= ((__float_as_uint(f.x) & 0x7F800000u) == 0x7F800000u) | ((__float_as_uint(f.y) & 0x7F800000u) == 0x7F800000u) |
                 ((__float_as_uint(f.z) & 0x7F800000u) == 0x7F800000u) | ((__float_as_uint(f.w) & 0x7F800000u) == 0x7F800000u);
        __stcs(reinterpret_cast<float4*>(dst + k), f);
      }
    } else {
      for (uint32_t k = lane; k < span; k += 32) {
        const float f = buf[k];
        buf[k] = 0.f;
        if (chk) bad |= (__float_as_uint(f) & 0x7F800000u) == 0x7F800000u;
        __stcs(dst + k, f);
      }
    }
    if (bad) fl |= FLAG_NONFINITE;
    __syncwarp();
  }
  if (cur >= 0) flush_flags(a, cur, fl, ck);
}

// ------------------------------------------------------------------------------- finalize
// One thread per stream: the reference's error precedence (codec.py:320-385, :235-252,
// tensor.py:27-36) from framing, CRC and validation flags; resets the accumulators.
__global__ void sif_dfinal_kernel(DecArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
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
