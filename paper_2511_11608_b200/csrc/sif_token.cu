// sif_token.cu -- fused encoder for token-sized IFs (sm_100a): one 128-thread CTA encodes
// one IF of <= 4096 elements (an LLM decode-step hidden state, 1 x 4096) from HBM to the
// finished .sif stream in ONE launch for the whole batch, with the IF held in shared
// memory throughout.  Every phase is short and wide (a batch of 1024 tokens is one wave of
// ~7 CTAs per SM, so the kernel time is the latency of one CTA):
//
//   load     the IF once (128-bit loads) into shared memory; thread t owns the 32
//            consecutive elements [32t, 32t+32) (16-byte slots swizzled by t & 7, so both
//            the coalesced fill and the per-thread reads are bank-conflict free); max key
//            for NaN/Inf (atkf.py:49-51)
//   tau      the k-th largest |x| key by a radix select over the IF with 8-bit digits and
//            one histogram per warp (levels whose bits are equal in every key, e.g. the
//            low half of bf16 data, are skipped) (atkf.py:71)
//   sort     elements with key >= tau, composite (|x| desc, plus first, flat index asc):
//            each warp sorts 128 of them in registers (bitonic network over shuffles), a
//            merge-path rank places every element (atkf.py:37-41; msplit.py:54-65)
//   ties     the r smallest splitmix64 hashes among the ties at tau (atkf.py:71-84)
//   blocks   per plane, the block cuts are the elements at plane ranks j * base of the
//            sorted order (msplit.py:68-80); block max / min = its first / last member
//            (quant.py:50-51)
//   members  each thread classifies its own candidates (kept test, block by comparison
//            with the cuts) and a packed per-block exclusive scan places them: block runs
//            in flat order = CSR order (msplit.py:92-95), no second sort
//   abq      DS sums of all blocks at once (quant.py:88-115); q* by the first violation
//   layout   .sif header / block metas (codec.py:283-317); pack: codes (quant.py:59-62),
//            MSB-first cols / codes (bitstream.py:6-30), row_ptr (msplit.py:97-100)
//   crc      CRC-32 of bytes [4, P-4) (codec.py:316), length and status
//
// The path takes lambda = 0, k >= 1 and at most KB blocks (the plan routes other IFs to the
// chunk pipeline); candidate sets larger than the register sort are sorted by a bitonic
// network in shared memory, or in the IF's global list area when larger still.  Output is
// byte-identical to the reference's.

#include "sif_post.cu"

namespace sif {

constexpr int KNT = 128;        // threads per token CTA
constexpr int KNW = KNT / 32;
constexpr int KT = 4096;        // max elements of a token-path IF
constexpr int KSORT = 1024;     // candidates sorted in shared memory
constexpr int KM = 512;         // candidates sorted by the register sort + merge
constexpr int KB = 8;           // max blocks (M+ + M-) on the token path

struct TokSh {
  uint4 raw[KNT][8];            // the IF: thread t's elements, slot j at [t][j ^ (t & 7)]
  union {
    uint32_t wh[KNW][256];      // radix levels of the tau select, one histogram per warp
    uint64_t srt[KSORT];        // then the sorted candidates, then the members (u32 flat
                                // indices, block runs back to back)
  } u;
  uint32_t whist[256];          // warp radix select of the tie hashes
  SelSh sh;
  uint32_t bsize[KB], brun[KB], bmin[KB], bmax[KB], q[KB], ckey[KB], cidx[KB];
  double vmin[KB], o64[KB], inv64[KB];
  double oq[KB][17], iq[KB][17];
  uint32_t S[KB][16];
  uint64_t meta[KB], bitc[KB], bitq[KB];
  uint64_t P, h_star;
  uint32_t ncand, G, E, tau, maxkey, kor, kand, tie_all, nnz0, nnz1, B, meff0, act[KB];
  uint32_t fd_digit, fd_above;
  uint64_t scan[40];
};

__device__ __forceinline__ uint32_t tok_raw(const TokSh& ts, uint32_t e) {
  const uint32_t t = e >> 5, j = (e >> 2) & 7u, k = e & 3u;
  const uint4 v = ts.raw[t][j ^ (t & 7u)];
  return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w;
}

// Bitonic sort (descending) of n composite keys at c[0 .. P), P = pow2 >= n, padding 0.
__device__ __forceinline__ void tok_sort(uint64_t* c, uint32_t n) {
  uint32_t P = 32;
  while (P < n) P <<= 1;
  for (uint32_t i = n + threadIdx.x; i < P; i += KNT) c[i] = 0ull;
  __syncthreads();
  for (uint32_t k = 2; k <= P; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t q = threadIdx.x; q < P / 2; q += KNT) {
        const uint32_t i = ((q & ~(j - 1)) << 1) | (q & (j - 1)), ix = i | j;
        const uint64_t x = c[i], y = c[ix];
        const bool desc = (i & k) == 0;
        if (desc ? (x < y) : (x > y)) { c[i] = y; c[ix] = x; }
      }
      __syncthreads();
    }
  }
}

// Sort (descending) n <= KM distinct nonzero composite keys at c[0 .. KM): warp w sorts
// c[128w .. 128w+128) in registers (4 per lane, bitonic network: exchanges over lane
// distance >= 4 by shuffles), then each element's final position is its run position plus
// the number of larger keys in the other three runs (binary searches).  Padding zeros land
// at positions >= n.
__device__ __forceinline__ void tok_sort512(uint64_t* c, uint32_t n) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (uint32_t i = n + tid; i < (uint32_t)KM; i += KNT) c[i] = 0ull;
  __syncthreads();
  uint64_t v[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) v[e] = c[w * 128 + 4 * lane + e];
#pragma unroll
  for (int k = 2; k <= 128; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 4) {
        const int lj = j >> 2;
        const bool lower = (lane & lj) == 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint64_t o = __shfl_xor_sync(0xFFFFFFFFu, v[e], lj);
          const bool desc = ((4 * lane + e) & k) == 0;
          const uint64_t hi = v[e] > o ? v[e] : o, lo = v[e] > o ? o : v[e];
          v[e] = (lower == desc) ? hi : lo;
        }
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (e & j) continue;
          const bool desc = ((4 * lane + e) & k) == 0;
          const uint64_t x = v[e], y = v[e | j];
          if (desc ? (x < y) : (x > y)) { v[e] = y; v[e | j] = x; }
        }
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) c[w * 128 + 4 * lane + e] = v[e];
  __syncthreads();
  uint32_t pos[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    uint32_t p = 4 * lane + e;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (r == w) continue;
      const uint64_t* run = c + r * 128;
      uint32_t lo = 0, hi = 128;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (run[mid] > v[e]) lo = mid + 1; else hi = mid;
      }
      p += lo;
    }
    pos[e] = p;
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < 4; ++e)
    if (pos[e] < (uint32_t)KM) c[pos[e]] = v[e];
  __syncthreads();
}

// The r-th smallest of the distinct 64-bit values val(i), i in [i0, i1), i1 - i0 <= 32 (one
// warp): every lane ranks its own value by comparing with all others.
template <class Val>
__device__ __forceinline__ uint64_t warp_select_small(uint32_t i0, uint32_t i1, uint64_t r, Val val) {
  const int lane = threadIdx.x & 31;
  const uint32_t m = i1 - i0;
  const uint64_t mine = (uint32_t)lane < m ? val(i0 + lane) : ~0ull;
  uint32_t rank = 0;
  for (uint32_t o = 0; o < m; ++o) {
    const uint64_t x = __shfl_sync(0xFFFFFFFFu, mine, o);
    rank += x < mine ? 1u : 0u;
  }
  const uint32_t hit = __ballot_sync(0xFFFFFFFFu, (uint32_t)lane < m && (uint64_t)rank + 1 == r);
  return __shfl_sync(0xFFFFFFFFu, mine, __ffs(hit) - 1);
}

__global__ void __launch_bounds__(KNT, 7) enc_token(EArgs a, const uint32_t* tok_list) {
  __shared__ TokSh ts;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int ifi = (int)tok_list[blockIdx.x];
  const IfInfo f = a.info[ifi];
  const uint32_t T = (uint32_t)f.T;
  const uint64_t kk = f.kk;
  const uint64_t seed = f.seed;

  prof_mark(a, ifi, 24);
  // ---- load (x read once from HBM)
  {
    uint32_t kor = 0, kand = 0xFFFFFFFFu, mk = 0;
    if (f.dtype == SIF_DTYPE_F32) {
      const uint4* x4 = reinterpret_cast<const uint4*>(f.x);
      for (uint32_t v = tid; v < KT / 4; v += KNT) {
        const uint32_t e = 4 * v;
        uint4 q = make_uint4(0, 0, 0, 0);
        if (e + 4 <= T) q = __ldcs(x4 + v);
        else if (e < T) {
          const uint32_t* x1 = reinterpret_cast<const uint32_t*>(f.x);
          q.x = x1[e];
          if (e + 1 < T) q.y = x1[e + 1];
          if (e + 2 < T) q.z = x1[e + 2];
        }
        const uint32_t t = e >> 5, j = (e >> 2) & 7u;
        ts.raw[t][j ^ (t & 7u)] = q;
      }
    } else {
      const uint4* x4 = reinterpret_cast<const uint4*>(f.x);
      for (uint32_t v = tid; v < KT / 8; v += KNT) {
        const uint32_t e = 8 * v;
        uint4 q = make_uint4(0, 0, 0, 0);
        if (e + 8 <= T) q = __ldcs(x4 + v);
        else if (e < T) {
          const unsigned short* x1 = reinterpret_cast<const unsigned short*>(f.x);
          uint32_t h[8] = {0, 0, 0, 0, 0, 0, 0, 0};
          for (uint32_t k = 0; k < 8 && e + k < T; ++k) h[k] = x1[e + k];
          q = make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16), h[6] | (h[7] << 16));
        }
        const uint32_t t = e >> 5, j = (e >> 2) & 7u;
        ts.raw[t][j ^ (t & 7u)] = make_uint4(q.x << 16, q.x & 0xFFFF0000u, q.y << 16, q.y & 0xFFFF0000u);
        ts.raw[t][(j + 1) ^ (t & 7u)] = make_uint4(q.z << 16, q.z & 0xFFFF0000u, q.w << 16, q.w & 0xFFFF0000u);
      }
    }
    if (tid == 0) { ts.kor = 0; ts.kand = 0xFFFFFFFFu; ts.maxkey = 0; ts.ncand = 0; ts.G = 0; }
    __syncthreads();
    for (int j = 0; j < 8; ++j) {
      const uint4 q = ts.raw[tid][j ^ (tid & 7)];
      const uint32_t v4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t e = 32u * tid + 4u * j + k;
        if (e < T) {
          const uint32_t key = v4[k] & 0x7FFFFFFFu;
          kor |= key;
          kand &= key;
          mk = max(mk, key);
        }
      }
    }
    kor = __reduce_or_sync(0xFFFFFFFFu, kor);
    kand = __reduce_and_sync(0xFFFFFFFFu, kand);
    mk = __reduce_max_sync(0xFFFFFFFFu, mk);
    if (lane == 0) { atomicOr(&ts.kor, kor); atomicAnd(&ts.kand, kand); atomicMax(&ts.maxkey, mk); }
    __syncthreads();
  }
  if (ts.maxkey >= kNonFiniteKey) {
    if (tid == 0) { a.status[ifi] = SIF_ERR_NONFINITE; a.out_len[ifi] = 0; }
    return;
  }

  prof_mark(a, ifi, 25);
  // ---- tau: the kk-th largest key; 8-bit digit levels (bits 23..30, 15..22, 7..14, 0..6),
  // levels whose bits do not vary skipped; one 256-bin histogram per warp
  uint32_t tau;
  {
    const uint32_t vary = ts.kor ^ ts.kand, cand = ts.kand;
    uint32_t r = (uint32_t)kk;
    uint32_t prefix = 0, mask = 0;
    const int shifts[4] = {23, 15, 7, 0}, widths[4] = {8, 8, 8, 7};
    uint32_t* wh = ts.u.wh[w];
    for (int lev = 0; lev < 4; ++lev) {
      const int shf = shifts[lev];
      const uint32_t nb = 1u << widths[lev];
      const uint32_t lmask = (nb - 1) << shf;
      if ((vary & lmask) == 0) {
        prefix |= cand & lmask;
        mask |= lmask;
        continue;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) wh[lane + 32 * k] = 0;
      __syncwarp();
      for (int j = 0; j < 8; ++j) {
        const uint4 q = ts.raw[tid][j ^ (tid & 7)];
        const uint32_t v4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t e = 32u * tid + 4u * j + k;
          const uint32_t key = v4[k] & 0x7FFFFFFFu;
          if (e < T && (key & mask) == prefix) atomicAdd(&wh[(key >> shf) & (nb - 1)], 1u);
        }
      }
      __syncthreads();
      if (w == 0) {  // digit holding rank r, from the top: lane l sums bins 255-8l .. 248-8l
        uint32_t v[8], sum = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t b = 255u - 8u * lane - j;
          v[j] = ts.u.wh[0][b] + ts.u.wh[1][b] + ts.u.wh[2][b] + ts.u.wh[3][b];
          sum += v[j];
        }
        const uint32_t inc = warp_incl_scan_u32(sum), exc = inc - sum;
        if (exc < r && r <= inc) {
          uint32_t acc = exc;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (acc < r && r <= acc + v[j]) { ts.fd_digit = 255u - 8u * lane - j; ts.fd_above = acc; }
            acc += v[j];
          }
        }
      }
      __syncthreads();
      prefix |= ts.fd_digit << shf;
      mask |= lmask;
      r -= ts.fd_above;
    }
    tau = prefix;
  }
  // tau == 0: fewer than kk nonzeros; every nonzero is kept (planes hold nonzeros only)
  const uint32_t tlo = tau > 0 ? tau : 1u;

  prof_mark(a, ifi, 26);
  // ---- candidates (key >= tau, nonzero) -> composite sort keys; cmask: this thread's
  // candidates (bit j = element 32 tid + j)
  uint32_t cmask = 0;
  uint64_t* srt;
  {
    uint32_t g = 0;
    for (int j = 0; j < 8; ++j) {
      const uint4 q = ts.raw[tid][j ^ (tid & 7)];
      const uint32_t v4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t e = 32u * tid + 4u * j + k;
        const uint32_t key = v4[k] & 0x7FFFFFFFu;
        cmask |= (e < T && key >= tlo ? 1u : 0u) << (4 * j + k);
        g += (e < T && key > tau && key >= tlo) ? 1u : 0u;
      }
    }
    uint32_t c = __popc(cmask);
    const uint32_t cin = warp_incl_scan_u32(c);
    g = __reduce_add_sync(0xFFFFFFFFu, g);
    uint32_t wbase = 0;
    if (lane == 31) wbase = atomicAdd(&ts.ncand, cin);
    if (lane == 0) atomicAdd(&ts.G, g);
    wbase = __shfl_sync(0xFFFFFFFFu, wbase, 31);
    __syncthreads();
    const uint32_t n = ts.ncand;
    // big tie sets (e.g. constant blocks): sort in the IF's global list area
    srt = n <= (uint32_t)KSORT ? ts.u.srt : reinterpret_cast<uint64_t*>(le(a, f));
    uint32_t p = wbase + cin - c;
    for (uint32_t m = cmask; m; m &= m - 1u) {
      const uint32_t jk = (uint32_t)(__ffs(m) - 1), e = 32u * tid + jk;
      const uint32_t v = tok_raw(ts, e);
      srt[p++] = ((uint64_t)(v & 0x7FFFFFFFu) << 33) | ((uint64_t)((v >> 31) ^ 1u) << 32) | (uint64_t)(~e);
    }
    __syncthreads();
    if (n <= (uint32_t)KM) tok_sort512(srt, n);
    else tok_sort(srt, n);
  }
  prof_mark(a, ifi, 27);
  const uint32_t n = ts.ncand, G = tau > 0 ? ts.G : n, E = n - G;
  auto key_at = [&](uint32_t p) -> uint32_t { return (uint32_t)(srt[p] >> 33); };
  auto idx_at = [&](uint32_t p) -> uint32_t { return ~(uint32_t)srt[p]; };

  // ---- ties at tau (warp 0): keep the r smallest splitmix64 hashes (atkf.py:37-41, :81-84)
  if (w == 0) {
    const uint64_t r_eq = tau > 0 ? kk - G : 0;
    const bool tie_all = tau == 0 || r_eq == E;
    uint64_t h_star = 0;
    if (!tie_all) {
      auto hv = [&](uint32_t i) -> uint64_t { return splitmix(seed, idx_at(i)); };
      h_star = E <= 32 ? warp_select_small(G, G + E, r_eq, hv)
                       : ~warp_select_range(ts.whist, G, G + E, r_eq, [&](uint32_t i) -> uint64_t { return ~hv(i); });
    }
    if (lane == 0) { ts.tie_all = tie_all ? 1u : 0u; ts.h_star = h_star; }
  }
  __syncthreads();
  const bool tie_all = ts.tie_all != 0;
  const uint64_t h_star = ts.h_star;
  auto kept_sorted = [&](uint32_t i) -> bool {
    return i < G || (i < n && (tie_all || splitmix(seed, idx_at(i)) <= h_star));
  };

  // ---- kept per sign; blocks by plane rank (msplit.py:68-80): in the sorted order a kept
  // element of plane s with rank r belongs to block min(r / base, meff - 1); its first
  // member is the block's cut and holds the block max, its last the block min
  // (quant.py:50-51).  Thread t walks the sorted entries [t E, t E + E); its starting plane
  // ranks come from a block scan of the per-thread kept counts (plus | minus << 16).
  {
    const uint32_t E = (n + KNT - 1) / KNT, i0 = tid * E, i1 = min(n, i0 + E);
    uint32_t kp = 0;
    for (uint32_t i = i0; i < i1; ++i)
      if (kept_sorted(i)) kp += ((srt[i] >> 32) & 1u) ? 1u : 0x10000u;
    uint32_t tot;
    const uint32_t ex = block_excl_scan_u32(kp, ts.sh.red, &tot);
    const uint32_t nnz[2] = {tot & 0xFFFFu, tot >> 16};
    const uint32_t mcfg[2] = {(uint32_t)a.m_plus, (uint32_t)a.m_minus};
    uint32_t meff[2], base[2];
    for (int sg = 0; sg < 2; ++sg) {
      meff[sg] = nnz[sg] < mcfg[sg] ? nnz[sg] : mcfg[sg];
      if (meff[sg] < 1) meff[sg] = 1;
      base[sg] = nnz[sg] / meff[sg];
    }
    const int B = (int)(meff[0] + meff[1]);
    if (tid < B) { ts.bmin[tid] = 0x7FFFFFFFu; ts.bmax[tid] = 0; ts.ckey[tid] = 0; ts.cidx[tid] = 0; }
    __syncthreads();
    uint32_t run[2] = {ex & 0xFFFFu, ex >> 16};
    for (uint32_t i = i0; i < i1; ++i) {
      if (!kept_sorted(i)) continue;
      const uint32_t sg = ((srt[i] >> 32) & 1u) ? 0u : 1u;
      const uint32_t r = run[sg]++;
      const uint32_t bs = base[sg], me_ = meff[sg];
      const uint32_t jl = min(r / bs, me_ - 1);
      const int b = (sg ? (int)meff[0] : 0) + (int)jl;
      const uint32_t last = jl + 1 < me_ ? (jl + 1) * bs - 1 : nnz[sg] - 1;
      if (r == jl * bs) { ts.bmax[b] = key_at(i); ts.ckey[b] = key_at(i); ts.cidx[b] = idx_at(i); }
      if (r == last) ts.bmin[b] = key_at(i);
    }
    if (tid == 0) {
      ts.nnz0 = nnz[0];
      ts.nnz1 = nnz[1];
      ts.B = (uint32_t)B;
      ts.meff0 = meff[0];
      uint32_t acc = 0;
      for (int b = 0; b < B; ++b) {
        const int sg = b < (int)meff[0] ? 0 : 1;
        const uint32_t m = meff[sg];
        const uint32_t j = sg ? (uint32_t)(b - (int)meff[0]) : (uint32_t)b;
        const uint32_t sz = nnz[sg] == 0 ? 0 : (j + 1 < m ? base[sg] : nnz[sg] - (m - 1) * base[sg]);
        ts.bsize[b] = sz;
        ts.brun[b] = acc;
        acc += sz;
      }
    }
  }
  __syncthreads();
  const int B = (int)ts.B;
  const int meff0 = (int)ts.meff0;
  prof_mark(a, ifi, 28);

  // ---- members: every thread classifies its own candidates in flat order; block runs
  // are placed by a packed exclusive scan of the per-thread block counts (16-bit fields,
  // blocks 0-3 in lo, 4-7 in hi), so each run is in flat order (CSR order, msplit.py:92-95)
  uint32_t* memv = reinterpret_cast<uint32_t*>(srt);  // srt is dead from here on
  {
    const int meff1 = B - meff0;
    auto block_of = [&](uint32_t e, uint32_t v) -> int {
      const uint32_t key = v & 0x7FFFFFFFu;
      if (tau > 0 && (key < tau || (key == tau && !tie_all && splitmix(seed, e) > h_star))) return -1;
      const bool plus = (v >> 31) == 0;
      const int b0 = plus ? 0 : meff0, nb = plus ? meff0 : meff1;
      int j = 0;
      for (int c = 1; c < nb; ++c) {  // at or after cut c in (key desc, index asc) order
        const uint32_t ck = ts.ckey[b0 + c], ci = ts.cidx[b0 + c];
        j += (key < ck || (key == ck && e >= ci)) ? 1 : 0;
      }
      return b0 + j;
    };
    // bc: block + 1 of this thread's candidate number o (0 = not kept), 4 bits each
    uint64_t lo = 0, hi = 0, bc0 = 0, bc1 = 0;
    uint32_t o = 0;
    for (uint32_t m = cmask; m; m &= m - 1u, ++o) {
      const uint32_t e = 32u * tid + (uint32_t)(__ffs(m) - 1);
      const int b = block_of(e, tok_raw(ts, e));
      if (b >= 4) hi += 1ull << (16 * (b - 4));
      else if (b >= 0) lo += 1ull << (16 * b);
      const uint64_t code = (uint64_t)(b + 1) << (4 * (o & 15u));
      if (o < 16) bc0 |= code; else bc1 |= code;
    }
    __syncthreads();  // every thread has read the sorted order (memv aliases it)
    uint64_t tot;
    uint64_t plo = block_excl_scan_u64(lo, ts.scan, &tot);
    uint64_t phi = block_excl_scan_u64(hi, ts.scan, &tot);
    o = 0;
    for (uint32_t m = cmask; m; m &= m - 1u, ++o) {
      const int b = (int)(((o < 16 ? bc0 : bc1) >> (4 * (o & 15u))) & 15u) - 1;
      if (b < 0) continue;
      const uint32_t e = 32u * tid + (uint32_t)(__ffs(m) - 1);
      uint32_t p;
      if (b >= 4) { p = (uint32_t)(phi >> (16 * (b - 4))) & 0xFFFFu; phi += 1ull << (16 * (b - 4)); }
      else { p = (uint32_t)(plo >> (16 * b)) & 0xFFFFu; plo += 1ull << (16 * b); }
      memv[ts.brun[b] + p] = e | ((uint32_t)b << 12);  // flat index (12 bits) and block
    }
  }
  __syncthreads();
  const uint32_t nk = ts.nnz0 + ts.nnz1;  // members, block runs back to back
  auto blk_of = [&](uint32_t i) -> int { return (int)(memv[i] >> 12); };
  auto mem_e = [&](uint32_t i) -> uint32_t { return memv[i] & 0xFFFu; };

  prof_mark(a, ifi, 29);
  // ---- ABQ (quant.py:88-115): all blocks at once, descending level by level while some
  // block is within delta
  const int qb = a.q_bit;
  const bool abq = a.mode != SIF_MODE_FIXED;
  for (int k = tid; k < B * 16; k += KNT) {
    const int b = k >> 4, q = (k & 15) + 1;
    ts.S[b][k & 15] = 0u;
    const double vmin = (double)__uint_as_float(ts.bmin[b]), vmax = (double)__uint_as_float(ts.bmax[b]);
    if (q <= qb) {
      const double o = __ddiv_rn(__dsub_rn(vmax, vmin), (double)((1u << q) - 1u));
      ts.oq[b][q] = o;
      ts.iq[b][q] = __drcp_rn(o);
    }
    if (q == 1) {
      ts.vmin[b] = vmin;
      ts.act[b] = (abq && qb >= 2 && ts.bsize[b] > 0 && ts.bmin[b] < ts.bmax[b]) ? 1u : 0u;
    }
  }
  __syncthreads();
  if (abq && qb >= 2) {
    const uint32_t lref = (1u << qb) - 1u;
    for (int qq = qb - 1; qq >= 1; --qq) {
      bool any = false;
      for (int b = 0; b < B; ++b) any |= ts.act[b] != 0;
      if (!any) break;
      const uint32_t lq = (1u << qq) - 1u;
      for (uint32_t i = tid; i < nk; i += KNT) {
        const int b = blk_of(i);
        if (!ts.act[b]) continue;
        const uint32_t key = tok_raw(ts, mem_e(i)) & 0x7FFFFFFFu;
        const double vmin = ts.vmin[b];
        const uint32_t r = quant_code(key, vmin, ts.oq[b][qb], ts.iq[b][qb], lref) >> (qb - qq);
        const uint32_t cq = quant_code(key, vmin, ts.oq[b][qq], ts.iq[b][qq], lq);
        const uint32_t d = r > cq ? r - cq : cq - r;
        if (d) atomicAdd(&ts.S[b][qq], d);
      }
      __syncthreads();
      if (tid < B && ts.act[tid])  // the first violation stops this block's descent
        ts.act[tid] = !(__ddiv_rn((double)ts.S[tid][qq], (double)ts.bsize[tid]) > a.delta) ? 1u : 0u;
      __syncthreads();
    }
  }

  // ---- layout (codec.py:176-181, :194-200, :269-317)
  if (tid < B) {
    const int b = tid;
    const int s = b < meff0 ? 0 : 1;
    const int j = s ? b - meff0 : b;
    const uint32_t nb = ts.bsize[b];
    const bool empty = nb == 0;
    const bool degen = !empty && ts.bmin[b] == ts.bmax[b];
    uint32_t q;
    if (!abq) q = a.fixed_q[(s ? a.m_plus : 0) + j];
    else if (empty) q = (uint32_t)qb;
    else if (degen) q = 1;
    else {
      q = (uint32_t)qb;
      for (int qq = qb - 1; qq >= 1; --qq) {
        const double ds = __ddiv_rn((double)ts.S[b][qq], (double)nb);
        if (ds > a.delta) break;
        q = (uint32_t)qq;
      }
    }
    ts.q[b] = q;
    const double vmin = (double)__uint_as_float(ts.bmin[b]), vmax = (double)__uint_as_float(ts.bmax[b]);
    const double o64 = (empty || degen) ? 1.0 : __ddiv_rn(__dsub_rn(vmax, vmin), (double)((1u << q) - 1u));
    ts.o64[b] = o64;
    ts.inv64[b] = __drcp_rn(o64);
    ts.vmin[b] = vmin;
  }
  __syncthreads();
  if (tid == 0) {
    uint64_t pos = kHeaderBytes + (abq ? 0ull : (uint64_t)B);
    for (int b = 0; b < B; ++b) {
      ts.meta[b] = pos;
      pos += kBlockMetaBytes + 4ull * ((uint64_t)f.N + 1ull);
      ts.bitc[b] = 8ull * pos;
      pos += ((uint64_t)ts.bsize[b] * f.cb + 7ull) / 8ull;
      ts.bitq[b] = 8ull * pos;
      pos += ((uint64_t)ts.bsize[b] * ts.q[b] + 7ull) / 8ull;
    }
    ts.P = pos + kCrcBytes;
  }
  __syncthreads();
  const uint64_t P = ts.P;
  if (P > f.cap) {
    if (tid == 0) { a.status[ifi] = SIF_ERR_CAPACITY; a.out_len[ifi] = P; }
    return;
  }
  uint8_t* out = f.out;
  {
    uint4* o4 = reinterpret_cast<uint4*>(out);
    const uint64_t n16 = P / 16;
    for (uint64_t z = tid; z < n16; z += KNT) o4[z] = make_uint4(0, 0, 0, 0);
    for (uint64_t z = n16 * 16 + tid; z < P; z += KNT) out[z] = 0;
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
    for (int b = tid; b < B; b += KNT) out[kHeaderBytes + b] = (uint8_t)ts.q[b];
  for (int b = tid; b < B; b += KNT) {
    const uint64_t o = ts.meta[b];
    out[o] = (uint8_t)ts.q[b];
    st_u32_le(out, o + 1, __float_as_uint(ts.bsize[b] == 0 ? 1.0f : __double2float_rn(ts.o64[b])));
    st_u32_le(out, o + 5, ts.bsize[b] == 0 ? 0u : ts.bmin[b]);
    st_u32_le(out, o + 9, ts.bsize[b]);
  }
  __syncthreads();

  prof_mark(a, ifi, 30);
  // ---- pack: thread per member of all blocks (bitstream.py:6-30), row_ptr (msplit.py:97-100)
  {
    FastDiv fk;
    fk.init(f.K);
    uint32_t* out32 = reinterpret_cast<uint32_t*>(out);
    const uint32_t cb = f.cb;
    for (uint32_t i = tid; i < nk; i += KNT) {
      const int b = blk_of(i);
      const uint32_t r0 = ts.brun[b], nb = ts.bsize[b], q = ts.q[b], m = i - r0;
      const uint64_t rp = ts.meta[b] + kBlockMetaBytes;
      const uint32_t ex = mem_e(i);
      const uint32_t row = fk.div(ex), col = ex - row * f.K;
      const int32_t prow = m > 0 ? (int32_t)fk.div(mem_e(i - 1)) : -1;
      for (int32_t r = prow + 1; r <= (int32_t)row; ++r) st_u32_le(out, rp + 4ull * (uint32_t)r, m);
      if (m + 1 == nb)  // rows after the last member hold nnz
        for (uint32_t r = row + 1; r <= f.N; ++r) st_u32_le(out, rp + 4ull * r, nb);
      if (cb == 8) out[(ts.bitc[b] >> 3) + m] = (uint8_t)col;
      else put_field(out32, ts.bitc[b] + (uint64_t)m * cb, col, cb);
      if (ts.bmin[b] != ts.bmax[b]) {
        const uint32_t code =
            quant_code(tok_raw(ts, ex) & 0x7FFFFFFFu, ts.vmin[b], ts.o64[b], ts.inv64[b], (1u << q) - 1u);
        if (q == 8) out[(ts.bitq[b] >> 3) + m] = (uint8_t)code;
        else put_field(out32, ts.bitq[b] + (uint64_t)m * q, code, q);
      }
    }
  }
  __syncthreads();

  prof_mark(a, ifi, 31);
  // ---- CRC of bytes [4, P-4)
  {
    uint32_t* t4 = reinterpret_cast<uint32_t*>(&ts.raw[0][0]);
    uint32_t* cstage = t4 + 1024;
    for (int k = tid; k < 1024; k += KNT) t4[k] = (&kCrcTab4[0][0])[k];
    __syncthreads();
    const uint32_t raw = crc_cta_pieces<KNT>(out, 4, P - 4, t4, ts.sh.red, cstage);
    if (tid == 0) {
      st_u32_le_bytes(out, P - 4, crc_finish(raw, P - 8));
      a.out_len[ifi] = P;
      a.status[ifi] = SIF_OK;
    }
  }
}

}  // namespace sif
