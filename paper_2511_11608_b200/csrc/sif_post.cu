// sif_post.cu -- per-IF encoder back end (sm_100a): ONE CTA takes an IF from its candidate
// list to the finished .sif stream.
//
// For IFs of a few thousand to a few hundred thousand elements (a ResNet split-point IF,
// 1024 x 196; the ResNet streams of a mixed batch) the chunk kernels after the stream pass
// (select, members, two ABQ passes, layout, pack, CRC: 7+ launches, chunk tables, cross-CTA
// atomics, the members array through L2) are replaced by one CTA per IF that loads the IF's
// candidates (written by enc_stream, |x| >= lo, ~1.1 k entries) into shared memory in flat
// order once and runs every later stage on them there:
//
//   load      digit histograms (global slot -> SMEM), candidates in flat order: the first
//             lcap in SMEM, the rest in the IF's spill area (a missed bracket re-streams the
//             IF first, keeping every nonzero)
//   select    select_if<0, PNT, true> (K3): tau, splitmix tie cut, lambda classes, kept
//             counts, MS cuts (atkf.py:37-96, msplit.py:54-80)
//   minmax    block min/max and last member (quant.py:50-51); block sizes come from the
//             select (msplit.py:68-80)
//   abq       DS sums at q_bit-1, then the lower levels for blocks still within delta
//             (quant.py:88-115)
//   layout    q*, offsets, header, block metas (codec.py:176-181, :269-317)
//   pack      flat-order tiles: each kept element's position in its block (CSR order =
//             flat order, msplit.py:92-95) from a per-tile scan, its col and code written
//             MSB-first at that position (bitstream.py:6-30), row_ptr transitions and tails
//             (msplit.py:97-100)
//   crc       CRC-32 of bytes [4, P-4) (codec.py:316), length and status
//
// Output is byte-identical to serialize(encode(x, cfg, seed)) of the reference.

#include "sif_enc.cu"

namespace sif {

constexpr int PNT = 1024;
constexpr int PNW = PNT / 32;
constexpr int kSmemSelectBytes = (2 * ND + 2 * HB + GCAP * 4 + 2 * GSM) * 4;
constexpr int TAG_SHIFT = 25;
constexpr uint32_t TAG_NONE = 0x7Fu;
constexpr uint32_t IDX_MASK = (1u << TAG_SHIFT) - 1u;
__device__ __forceinline__ int tag_blk(uint32_t y) {
  const uint32_t t = y >> TAG_SHIFT;
  return t == TAG_NONE ? -1 : (int)t;
}

struct PostSh {
  K3Sh k3;
  KeptCtx kc;
  uint32_t red[2 * PNW + 2];
  uint32_t wcnt[PNW][MAXB];
  int32_t wlast[PNW][MAXB];
  uint32_t bsize[MAXB], brun[MAXB], bfill[MAXB], bmin[MAXB], bmax[MAXB], q[MAXB], act[MAXB];
  int32_t blast[MAXB];
  double vmin[MAXB], o64[MAXB], inv64[MAXB];
  unsigned long long S[MAXB][16];
  uint64_t meta[MAXB], bitc[MAXB], bitq[MAXB];
  uint64_t P;
  uint32_t ncand, err, cursor;
};

// ABQ scales: shared memory that is free once the select is done
struct PostAbq {
  double oq[MAXB][17], iq[MAXB][17];
};

// Warp-uniform pass over the n list entries (4 per thread in flight; every lane calls f,
// invalid ones with valid = false, so f may use warp collectives).
template <class F>
__device__ __forceinline__ void post_pass(const List& L, uint32_t n, F f) {
  for (uint32_t i0 = 0; i0 < n; i0 += 4 * PNT) {
    uint2 e[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t i = i0 + threadIdx.x + k * PNT;
      e[k] = i < n ? L.get(i) : make_uint2(0, 0);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) f(e[k], i0 + threadIdx.x + k * PNT < n);
  }
}

// MSB-first w-bit field (w <= 32) at absolute bit `bit` of a zeroed, word-aligned buffer.
__device__ __forceinline__ void put_field(uint32_t* out32, uint64_t bit, uint32_t val, uint32_t w) {
  const uint64_t W = bit >> 5;
  const uint32_t sh = (uint32_t)(bit & 31u);
  const uint64_t x = (uint64_t)val << (64u - w - sh);
  const uint32_t hi = (uint32_t)(x >> 32), lo = (uint32_t)x;
  if (hi) atomicOr(out32 + W, bswap32(hi));
  if (sh + w > 32u && lo) atomicOr(out32 + W + 1, bswap32(lo));
}

__global__ void __launch_bounds__(PNT, 1) enc_post(EArgs a, const uint32_t* post_list, uint32_t lcap) {
  extern __shared__ __align__(16) uint8_t dsm_raw[];
  uint32_t* dsm = reinterpret_cast<uint32_t*>(dsm_raw);
  __shared__ PostSh ps;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  const int ifi = (int)post_list[blockIdx.x];
  const IfInfo f = a.info[ifi];
  IfSt& st = a.st[ifi];
  const uint64_t kk = f.kk;
  uint32_t* hist = dsm;
  uint2* lsm = reinterpret_cast<uint2*>(dsm_raw + kSmemSelectBytes);
  prof_mark(a, ifi, 16);

  // ---- load: histogram and candidates (flat order); NaN/Inf; a missed bracket re-streams
  if (st.maxkey >= kNonFiniteKey) {  // atkf.py:49-51
    zero_hist(a, f);
    if (tid == 0) { st.err = E_NONFINITE; a.status[ifi] = SIF_ERR_NONFINITE; a.out_len[ifi] = 0; }
    return;
  }
  uint32_t lo = st.lo, lo_neg = st.lo_neg;
  const uint32_t nunits = f.nch * UNITS;
  const uint64_t u0 = (uint64_t)f.ch0 * UNITS;
  if (kk > 0 && st.cnt_lo < kk && lo > 1) {
    // bracket missed: every nonzero is a candidate; units re-streamed by all warps (list
    // order is free: u_off / u_cnt record each unit's segment)
    lo = 1;
    lo_neg = 1;
    for (int k = tid; k < 2 * ND; k += PNT) hist[k] = 0;
    if (tid == 0) ps.cursor = 0;
    __syncthreads();
    uint2* stage = reinterpret_cast<uint2*>(dsm + 2 * ND) + w * UE;
    uint32_t mk = 0, clo = 0, dmin = 0, dmax = 0;
    for (uint32_t u = (uint32_t)w; u < nunits; u += PNW) {
      const uint32_t c = f.ch0 + u / UNITS;
      uint32_t e0, n;
      unit_span(a, f, c, u % UNITS, e0, n);
      uint32_t cnt = 0;
      if (n) {
        Raw r;
        load_unit(f.x, f.dtype, e0, n, r);
        cnt = classify_any(f.dtype, r, e0, n, lo, lo_neg, false, stage, clo);
      }
      uint32_t off = 0;
      if (lane == 0) {
        off = atomicAdd(&ps.cursor, cnt);
        a.u_off[u0 + u] = off;
        a.u_cnt[u0 + u] = cnt;
      }
      off = __shfl_sync(0xFFFFFFFFu, off, 0);
      __syncwarp();
      emit_unit(stage, cnt, le(a, f) + off, hist, mk, dmin, dmax);
      __syncwarp();
    }
    __syncthreads();
    if (tid == 0) { st.lo = 1; st.lo_neg = 1; st.cnt_lo = ps.cursor; st.ncand = ps.cursor; }
    zero_hist(a, f);
  } else {
    const uint4* gh = reinterpret_cast<const uint4*>(a.hist + (uint64_t)f.hslot * 2 * ND);
    uint4* h4 = reinterpret_cast<uint4*>(hist);
    for (int k = tid; k < 2 * ND / 4; k += PNT) h4[k] = __ldcg(gh + k);
    __syncthreads();
    zero_hist(a, f);  // the slot starts zeroed for the next run
  }
  __syncthreads();
  // flat order: exclusive prefix of the unit counts (units in chunk order), then a warp per
  // unit copies its segment; the first lcap entries land in shared memory
  const List LP{lsm, reinterpret_cast<uint2*>(a.ws + f.sp_off), lcap};
  {
    // units of the IF in chunk order: exclusive prefix of their counts (scratch after the
    // histogram), then a warp per unit copies its segment, coalesced
    uint32_t* upre = dsm + 2 * ND;
    const uint2* src = le(a, f);
    uint32_t run = 0;
    for (uint32_t b0 = 0; b0 < nunits; b0 += PNT) {
      const uint32_t u = b0 + tid;
      const uint32_t cnt = u < nunits ? a.u_cnt[u0 + u] : 0u;
      uint32_t tot;
      const uint32_t ex = block_excl_scan_u32(cnt, ps.red, &tot);
      if (u < nunits) upre[u] = run + ex;
      run += tot;
    }
    if (tid == 0) { ps.ncand = run; st.ncand = run; }
    __syncthreads();
    for (uint32_t u = (uint32_t)w; u < nunits; u += PNW) {
      const uint32_t cnt = a.u_cnt[u0 + u], off = a.u_off[u0 + u], dst = upre[u];
      for (uint32_t j0 = 0; j0 < cnt; j0 += 256) {
        uint2 ev[8];
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          const uint32_t j = j0 + 32 * h + lane;
          ev[h] = j < cnt ? __ldcs(src + off + j) : make_uint2(0, 0);  // read once: evict-first
        }
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          const uint32_t j = j0 + 32 * h + lane;
          if (j < cnt) LP.set(dst + j, ev[h].x, ev[h].y);
        }
      }
    }
  }
  __syncthreads();
  prof_mark(a, ifi, 17);

  // ---- select (K3)
  select_if<0, PNT, true>(a, ifi, dsm, ps.k3, &LP);
  __syncthreads();
  prof_mark(a, ifi, 18);

  // ---- block sizes (from the select), min / max / last member (quant.py:50-51)
  const int B = (int)st.B;
  const int meff0 = (int)st.meff0;
  const uint32_t ncand = ps.ncand;
  if (tid == 0) {
    load_kept_ctx(ps.kc, st, f.seed);
    uint32_t acc = 0;
    for (int b = 0; b < B; ++b) {
      const int s = b < meff0 ? 0 : 1;
      const uint64_t m = s ? (uint64_t)(B - meff0) : (uint64_t)meff0;
      const uint64_t j = s ? (uint64_t)(b - meff0) : (uint64_t)b;
      const uint64_t n = st.nnz[s];
      const uint64_t sz = n == 0 ? 0 : (j + 1 < m ? st.base[s] : n - (m - 1) * st.base[s]);
      ps.bsize[b] = (uint32_t)sz;
      ps.brun[b] = acc;
      acc += (uint32_t)sz;
      ps.bfill[b] = 0;
      ps.bmin[b] = 0x7FFFFFFFu;
      ps.bmax[b] = 0;
      ps.blast[b] = -1;
    }
  }
  __syncthreads();
  // tag pass: the kept test and block id once per candidate (the block id rides in the
  // top 7 bits of the flat index, TAG_NONE = not kept; post IFs have < 2^25 elements), and
  // block min / max
  {
    const bool few = B <= 8;
    for (uint32_t i0 = 0; i0 < ncand; i0 += PNT) {
      const uint32_t i = i0 + tid;
      const bool v = i < ncand;
      uint2 e = v ? LP.get(i) : make_uint2(0, 0);
      const int blk = (v && ps.kc.kept(e.x, e.y)) ? ps.kc.block_of(e.x, e.y) : -1;
      if (v) LP.set(i, e.x, e.y | ((blk >= 0 ? (uint32_t)blk : TAG_NONE) << TAG_SHIFT));
      const uint32_t key = e.x & 0x7FFFFFFFu;
      if (few) {
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          if (b < B) {
            const bool in = blk == b;
            const uint32_t mn = __reduce_min_sync(0xFFFFFFFFu, in ? key : 0x7FFFFFFFu);
            const uint32_t mx = __reduce_max_sync(0xFFFFFFFFu, in ? key : 0u);
            if (lane == b && mn <= mx) {
              atomicMin(&ps.bmin[b], mn);
              atomicMax(&ps.bmax[b], mx);
            }
          }
        }
      } else {
        const uint32_t peers = __match_any_sync(0xFFFFFFFFu, blk);
        if (blk >= 0) {
          const uint32_t mn = __reduce_min_sync(peers, key), mx = __reduce_max_sync(peers, key);
          if ((peers & lt) == 0) {
            atomicMin(&ps.bmin[blk], mn);
            atomicMax(&ps.bmax[blk], mx);
          }
        }
      }
    }
  }
  __syncthreads();
  prof_mark(a, ifi, 19);

  // ---- ABQ (K5): S[b][q] = sum |code_qbit >> (qbit - q) - code_q| (quant.py:88-115)
  PostAbq& pa = *reinterpret_cast<PostAbq*>(dsm_raw);
  const int qb = a.q_bit;
  const bool abq = a.mode != SIF_MODE_FIXED;
  for (int k = tid; k < B * 16; k += PNT) {
    const int b = k >> 4, q = (k & 15) + 1;
    ps.S[b][k & 15] = 0ull;
    const double vmin = (double)__uint_as_float(ps.bmin[b]), vmax = (double)__uint_as_float(ps.bmax[b]);
    if (q <= qb) {
      const double o = __ddiv_rn(__dsub_rn(vmax, vmin), (double)((1u << q) - 1u));
      pa.oq[b][q] = o;
      pa.iq[b][q] = __drcp_rn(o);
    }
    if (q == 1) {
      ps.vmin[b] = vmin;
      ps.act[b] = (abq && qb >= 2 && ps.bsize[b] > 0 && ps.bmin[b] < ps.bmax[b]) ? 1u : 0u;
    }
  }
  __syncthreads();
  if (abq && qb >= 2) {
    const uint32_t lref = (1u << qb) - 1u, l1 = (1u << (qb - 1)) - 1u;
    // pass A: q_bit - 1 for every non-degenerate block
    {
      const bool few = B <= 8;
      unsigned long long accb[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      post_pass(LP, ncand, [&](uint2 e, bool v) {
        int blk = v ? tag_blk(e.y) : -1;
        if (blk >= 0 && !ps.act[blk]) blk = -1;
        uint32_t d = 0;
        if (blk >= 0) {
          const uint32_t key = e.x & 0x7FFFFFFFu;
          const double vmin = ps.vmin[blk];
          const uint32_t r = quant_code(key, vmin, pa.oq[blk][qb], pa.iq[blk][qb], lref) >> 1;
          const uint32_t cq = quant_code(key, vmin, pa.oq[blk][qb - 1], pa.iq[blk][qb - 1], l1);
          d = r > cq ? r - cq : cq - r;
        }
        if (few) {
#pragma unroll
          for (int b = 0; b < 8; ++b)
            if (b < B) accb[b] += __reduce_add_sync(0xFFFFFFFFu, blk == b ? d : 0u);
        } else {
          const uint32_t peers = __match_any_sync(0xFFFFFFFFu, blk);
          if (blk >= 0) {
            const uint32_t sum = __reduce_add_sync(peers, d);
            if ((peers & lt) == 0 && sum) atomicAdd(&ps.S[blk][qb - 1], (unsigned long long)sum);
          }
        }
      });
      if (few && lane == 0) {
#pragma unroll
        for (int b = 0; b < 8; ++b)
          if (b < B && accb[b]) atomicAdd(&ps.S[b][qb - 1], accb[b]);
      }
    }
    __syncthreads();
    // pass B: every q < q_bit - 1 for blocks whose q_bit - 1 distortion is within delta
    if (tid < B && ps.act[tid])
      ps.act[tid] = !(__ddiv_rn((double)ps.S[tid][qb - 1], (double)ps.bsize[tid]) > a.delta) ? 1u : 0u;
    __syncthreads();
    bool any = false;
    for (int b = 0; b < B; ++b) any |= ps.act[b] != 0;
    if (qb >= 3 && any) {
      post_pass(LP, ncand, [&](uint2 e, bool v) {
        int blk = v ? tag_blk(e.y) : -1;
        if (blk >= 0 && !ps.act[blk]) blk = -1;
        const uint32_t peers = __match_any_sync(0xFFFFFFFFu, blk);
        if (blk < 0) return;
        const uint32_t key = e.x & 0x7FFFFFFFu;
        const double vmin = ps.vmin[blk];
        const uint32_t cr = quant_code(key, vmin, pa.oq[blk][qb], pa.iq[blk][qb], lref);
        for (int q = 1; q < qb - 1; ++q) {
          const uint32_t cq = quant_code(key, vmin, pa.oq[blk][q], pa.iq[blk][q], (1u << q) - 1u);
          const uint32_t r = cr >> (qb - q);
          const uint32_t sum = __reduce_add_sync(peers, r > cq ? r - cq : cq - r);
          if ((peers & lt) == 0 && sum) atomicAdd(&ps.S[blk][q], (unsigned long long)sum);
        }
      });
    }
    __syncthreads();
  }
  prof_mark(a, ifi, 20);

  // ---- layout (K6): q*, o, offsets (quant.py:102-115; codec.py:176-181, :194-200, :269-317)
  if (tid < B) {
    const int b = tid;
    const int s = b < meff0 ? 0 : 1;
    const int j = s ? b - meff0 : b;
    const uint32_t n = ps.bsize[b];
    const bool empty = n == 0;
    const bool degen = !empty && ps.bmin[b] == ps.bmax[b];
    uint32_t q;
    if (!abq) q = a.fixed_q[(s ? a.m_plus : 0) + j];
    else if (empty) q = (uint32_t)qb;
    else if (degen) q = 1;
    else {
      q = (uint32_t)qb;
      for (int qq = qb - 1; qq >= 1; --qq) {
        const double ds = __ddiv_rn((double)ps.S[b][qq], (double)n);
        if (ds > a.delta) break;  // the first violation stops the descent
        q = (uint32_t)qq;
      }
    }
    ps.q[b] = q;
    const double vmin = (double)__uint_as_float(ps.bmin[b]), vmax = (double)__uint_as_float(ps.bmax[b]);
    const double o64 = (empty || degen) ? 1.0 : __ddiv_rn(__dsub_rn(vmax, vmin), (double)((1u << q) - 1u));
    ps.o64[b] = o64;
    ps.inv64[b] = __drcp_rn(o64);
    ps.vmin[b] = vmin;
  }
  __syncthreads();
  if (tid == 0) {
    uint64_t pos = kHeaderBytes + (abq ? 0ull : (uint64_t)B);
    for (int b = 0; b < B; ++b) {
      ps.meta[b] = pos;
      pos += kBlockMetaBytes + 4ull * ((uint64_t)f.N + 1ull);
      ps.bitc[b] = 8ull * pos;
      pos += ((uint64_t)ps.bsize[b] * f.cb + 7ull) / 8ull;
      ps.bitq[b] = 8ull * pos;
      pos += ((uint64_t)ps.bsize[b] * ps.q[b] + 7ull) / 8ull;
    }
    ps.P = pos + kCrcBytes;
    ps.err = ps.P > f.cap ? E_CAPACITY : E_NONE;
  }
  __syncthreads();
  const uint64_t P = ps.P;
  if (ps.err) {
    if (tid == 0) { st.err = E_CAPACITY; a.status[ifi] = SIF_ERR_CAPACITY; a.out_len[ifi] = P; }
    return;
  }
  uint8_t* out = f.out;
  {  // zero [0, P): packed fields are OR-ed into place
    uint4* o4 = reinterpret_cast<uint4*>(out);
    const uint64_t n16 = P / 16;
    for (uint64_t z = tid; z < n16; z += PNT) o4[z] = make_uint4(0, 0, 0, 0);
    for (uint64_t z = n16 * 16 + tid; z < P; z += PNT) out[z] = 0;
  }
  __syncthreads();
  if (tid == 0) {
    uint8_t h[32];
    h[0] = 'S'; h[1] = 'I'; h[2] = 'F'; h[3] = '1';
    h[4] = 1; h[5] = 0;
    for (int k = 0; k < 4; ++k) { h[6 + k] = (uint8_t)(f.N >> (8 * k)); h[10 + k] = (uint8_t)(f.K >> (8 * k)); }
    const uint32_t s32 = __float_as_uint(__double2float_rn(a.s));
    const uint32_t l32 = __float_as_uint(__double2float_rn(a.lam));
    const uint32_t d32 = __float_as_uint(__double2float_rn(a.delta));
    for (int k = 0; k < 4; ++k) {
      h[14 + k] = (uint8_t)(s32 >> (8 * k));
      h[18 + k] = (uint8_t)(l32 >> (8 * k));
      h[23 + k] = (uint8_t)(d32 >> (8 * k));
    }
    h[22] = (uint8_t)qb;
    h[27] = (uint8_t)a.mode;
    const uint32_t m0 = (uint32_t)meff0, m1 = (uint32_t)(B - meff0);
    h[28] = (uint8_t)m0; h[29] = (uint8_t)(m0 >> 8);
    h[30] = (uint8_t)m1; h[31] = (uint8_t)(m1 >> 8);
    for (int k = 0; k < 32; ++k) out[k] = h[k];
  }
  if (!abq)
    for (int b = tid; b < B; b += PNT) out[kHeaderBytes + b] = (uint8_t)ps.q[b];
  for (int b = tid; b < B; b += PNT) {
    const uint64_t o = ps.meta[b];
    out[o] = (uint8_t)ps.q[b];
    st_u32_le(out, o + 1, __float_as_uint(ps.bsize[b] == 0 ? 1.0f : __double2float_rn(ps.o64[b])));
    st_u32_le(out, o + 5, ps.bsize[b] == 0 ? 0u : ps.bmin[b]);
    st_u32_le(out, o + 9, ps.bsize[b]);
  }
  __syncthreads();
  prof_mark(a, ifi, 21);

  // ---- pack (K7): flat-order tiles of PNT entries; position of each member in its block
  // run from the tile scan (per warp and block: count and last row), then col / code fields
  // (bitstream.py:6-30) and the row_ptr entries of the rows this member opens
  {
    FastDiv fk;
    fk.init(f.K);
    uint32_t* out32 = reinterpret_cast<uint32_t*>(out);
    const uint32_t cb = f.cb;
    for (uint32_t i0 = 0; i0 < ncand; i0 += PNT) {
      const uint32_t i = i0 + tid;
      const bool v = i < ncand;
      const uint2 e0 = v ? LP.get(i) : make_uint2(0, 0);
      const int blk = v ? tag_blk(e0.y) : -1;
      const uint2 e = make_uint2(e0.x, e0.y & IDX_MASK);
      const uint32_t row = fk.div(e.y);
      const uint32_t peers = __match_any_sync(0xFFFFFFFFu, blk);
      const uint32_t below = peers & lt;
      const int pred = below ? 31 - __clz(below) : lane;
      const int32_t prow_w = __shfl_sync(0xFFFFFFFFu, (int32_t)row, pred);
      for (int b = lane; b < B; b += 32) { ps.wcnt[w][b] = 0; ps.wlast[w][b] = -1; }
      __syncwarp();
      if (blk >= 0 && lane == 31 - __clz(peers)) { ps.wcnt[w][blk] = __popc(peers); ps.wlast[w][blk] = (int32_t)row; }
      __syncthreads();
      if (tid < B) {
        uint32_t run = ps.bfill[tid];
        int32_t last = ps.blast[tid];
        for (int k = 0; k < PNW; ++k) {
          const uint32_t c = ps.wcnt[k][tid];
          const int32_t l = ps.wlast[k][tid];
          ps.wcnt[k][tid] = run;
          ps.wlast[k][tid] = last;
          run += c;
          if (c) last = l;
        }
        ps.bfill[tid] = run;
        ps.blast[tid] = last;
      }
      __syncthreads();
      if (blk >= 0) {
        const uint32_t pos = ps.wcnt[w][blk] + __popc(below);
        const int32_t prow = below ? prow_w : ps.wlast[w][blk];
        const uint64_t rp = ps.meta[blk] + kBlockMetaBytes;
        for (int32_t r = prow + 1; r <= (int32_t)row; ++r) st_u32_le(out, rp + 4ull * (uint32_t)r, pos);
        const uint32_t col = e.y - row * f.K;
        if (cb == 8) out[(ps.bitc[blk] >> 3) + pos] = (uint8_t)col;
        else put_field(out32, ps.bitc[blk] + (uint64_t)pos * cb, col, cb);
        if (ps.bmin[blk] != ps.bmax[blk]) {
          const uint32_t q = ps.q[blk];
          const uint32_t code = quant_code(e.x & 0x7FFFFFFFu, ps.vmin[blk], ps.o64[blk], ps.inv64[blk], (1u << q) - 1u);
          if (q == 8) out[(ps.bitq[blk] >> 3) + pos] = (uint8_t)code;
          else put_field(out32, ps.bitq[blk] + (uint64_t)pos * q, code, q);
        }
      }
      __syncthreads();
    }
    // row_ptr tails: rows after the block's last member hold nnz (msplit.py:97-100)
    for (int b = 0; b < B; ++b) {
      const uint32_t nb = ps.bsize[b];
      if (nb == 0) continue;
      const uint64_t rp = ps.meta[b] + kBlockMetaBytes;
      for (uint32_t r = (uint32_t)(ps.blast[b] + 1) + tid; r <= f.N; r += PNT) st_u32_le(out, rp + 4ull * r, nb);
    }
  }
  __syncthreads();
  prof_mark(a, ifi, 22);

  // ---- CRC (K8) of bytes [4, P-4), from L2
  {
    uint32_t* t4 = dsm;
    uint32_t* cstage = dsm + 1024;
    for (int k = tid; k < 1024; k += PNT) t4[k] = (&kCrcTab4[0][0])[k];
    __syncthreads();
    const uint32_t raw = crc_cta_staged<PNT>(out, 4, P - 4, t4, ps.red, cstage);
    if (tid == 0) {
      st_u32_le_bytes(out, P - 4, crc_finish(raw, P - 8));
      a.out_len[ifi] = P;
      a.status[ifi] = SIF_OK;
    }
  }
  prof_mark(a, ifi, 23);
}

}  // namespace sif
