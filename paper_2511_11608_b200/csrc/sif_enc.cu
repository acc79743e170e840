// sif_enc.cu -- B200 (sm_100a) encoder for the SLICER IF codec: a chunk-parallel pipeline.
//
// A batch of IFs is cut into chunks of CH elements (flat order).  Every stage is one
// kernel over either all chunks of the batch (persistent CTAs, grid = k x 148 SMs) or one
// CTA per IF, so each stage fills the whole GPU whatever the IF sizes are:
//
//   K1 enc_prep     (per IF)    zero per-IF accumulators; sampled bracket lo for tau
//   K2 enc_stream   (chunks)    the only pass over the IF in HBM: NaN/Inf check, stable
//                               compaction of candidates |x| >= lo into the IF's list
//                               (chunk segments in flat order), per-sign 12-bit digit
//                               histograms of the candidates
//   K3 enc_select   (per IF)    tau + tie cut (atkf.py:37-41, :71-84), kept counts per
//                               sign, MS cut elements (msplit.py:54-80).  Digit histogram ->
//                               gather of one digit bin -> exact select inside the bin
//   K4 enc_members  (chunks)    kept test, block id, stable regroup of each chunk segment
//                               by block (CSR order inside a block = flat order), block
//                               min/max (quant.py:50-51), per-chunk block counts
//   K5 enc_abq      (chunks)    ABQ distortion sums for every candidate q (quant.py:88-115)
//   K6 enc_layout   (per IF)    q* per block, .sif layout, header/meta, chunk prefixes,
//                               row_ptr tails (codec.py:269-317, msplit.py:97-100)
//   K7 enc_pack     (chunks)    codes (quant.py:59-62), row_ptr transitions, MSB-first
//                               word assembly of cols and codes (bitstream.py:6-30)
//   K8 enc_crc      (per IF)    CRC-32 over bytes [4, P-4) (codec.py:316), lengths, status
//
// The only HBM pass over the input is K2; candidate lists (|x| >= lo, ~k_keep entries)
// live in a workspace that mostly stays L2-resident between stages.  Output is
// byte-identical to serialize(encode(x, cfg, seed)) of the reference.

#include <math.h>
#include <stdint.h>

#include "sif_common.cuh"

namespace sif {

constexpr int CH = 4096;           // elements per chunk
constexpr int UNITS = 8;           // warp-streamed units per chunk
constexpr int UE = CH / UNITS;     // elements per unit
constexpr int CNT = 256;           // threads of chunk kernels
constexpr int DSH = 19;            // digit = |x| key >> 19 (12 bits)
constexpr int ND = 4096;           // digits per sign
constexpr int MAXB = 64;           // max effective blocks (M+ + M-) per IF (two per lane in the chunk kernels)
constexpr int MAXREG = 32;         // gather regions per IF (one per lane in enc_gather)
constexpr int SNT = 512;           // threads of the per-IF select kernel
constexpr int HB = 2048;           // radix histogram bins inside select_exact
constexpr int GCAP = 1024;         // in-SMEM exact ranking capacity
constexpr int GSM = 4096;          // gather list entries held in SMEM (K3)
constexpr uint32_t kInfKey = 0xFFFFFFFFu;

enum : uint32_t {
  F_KEEP_NONE = 1u, F_ONLY_NONZERO = 2u, F_ZERO_MODE = 4u, F_USE_CLS = 8u, F_TIE_ALL = 16u
};
enum : uint32_t { E_NONE = 0u, E_NONFINITE = 1u, E_CAPACITY = 2u };
// PATH_PIPE: every stage is a chunk / per-IF kernel of this file.  PATH_POST: prep and
// stream as PATH_PIPE, then one CTA per IF runs select .. CRC with the candidate list in
// shared memory (enc_post, sif_post.cu).
// PATH_TOKEN: the whole encode of a token-sized IF in one CTA (enc_token, sif_token.cu).
enum : uint32_t { PATH_PIPE = 0u, PATH_POST = 1u, PATH_TOKEN = 2u };

// Static per-IF description, built on the host (sif_enc_upload).
struct IfInfo {
  const void* x;
  uint8_t* out;
  uint64_t cap, seed, T, kk;
  uint32_t N, K, cb, dtype;
  uint32_t ch0, nch;
  int32_t hslot;
  uint32_t path;      // PATH_PIPE / PATH_POST
  uint64_t list_off;  // workspace byte offset of the candidate list: uint2[T]
  uint64_t gat_off;   // gather spill / member slots: uint2[T]
  uint64_t sp_off;    // PATH_POST: the candidates beyond enc_post's shared-memory part, uint2[T]
};

// Dynamic per-IF state (device).
struct IfSt {
  uint32_t lo, lo_neg, ncand, maxkey;
  uint32_t cnt_lo, err, flags, tau_key;
  uint64_t ck_star, h_star;
  double tau, tau_p, tau_m;
  uint32_t B, ncut0, ncut, meff0;
  uint64_t nnz[2], base[2];
  uint32_t cut_key[MAXB], cut_idx[MAXB];
  uint32_t bmin[MAXB], bmax[MAXB], q[MAXB], pad1;
  uint64_t bn[MAXB];
  uint64_t S[MAXB * 16];
  double o64[MAXB], inv64[MAXB];
  uint64_t off_meta[MAXB], bit_cols[MAXB], bit_codes[MAXB];
  uint64_t P;
  uint32_t crc_acc, seg_done;
  uint32_t bcount[MAXB];  // block member totals (K4 atomics)
  // multi-kernel select state (enc_select<1|2>, enc_gather<1|2>)
  uint32_t sel_phase;     // 0 done, 1 needs the tau-bin gather, 2 needs the cut-bin gather,
                          // 4 resolved by enc_select_tiny
  int32_t dtau;
  uint64_t rt, cnt_nz;
  uint32_t nA, pend_n, nreg, sel_lo;
  uint32_t pend_s[MAXB], pend_d[MAXB], pend_r[MAXB], pend_ci[MAXB], pend_reg[MAXB];
  uint32_t reg_off[MAXB], reg_cnt[MAXB], reg_key[MAXB];
  uint32_t nreg_pre, reg_first, pre_end;  // regions filled by enc_gather<1>, first for <2>, end offset
};

struct EArgs {
  const IfInfo* info;
  IfSt* st;
  int n, nch, maxb, atkf_only;
  const uint32_t* ch_if;
  const uint32_t* ch_e0;
  uint32_t* u_off;     // [nch][UNITS] list offset of each unit's candidates
  uint32_t* u_cnt;     // [nch][UNITS]
  uint32_t* ch_bcnt;   // [nch][maxb]
  uint32_t* ch_bpre;   // [nch][maxb]
  uint32_t* ch_brs;    // [nch][maxb] start of the block's run inside the chunk's member slot
  int32_t* ch_blast;   // [nch][maxb] row of the block's last member in the chunk, -1 if none
  int32_t* ch_bprev;   // [nch][maxb] row of the block's last member in earlier chunks
  uint32_t* hist;      // [nhist][2][ND]
  uint8_t* ws;
  double s, lam, delta;
  int m_plus, m_minus, q_bit, mode;
  const uint8_t* fixed_q;
  uint64_t* out_len;
  int32_t* status;
  int64_t* kept_out;
  const uint64_t* kept_off;
  double* tau3;
  const uint32_t* seg_base;  // [n+1] prefix of CRC segments per IF
  uint64_t* prof;            // optional phase timestamps (32 per IF: enc_select 0-8, enc_post 16-23; debug)
  uint32_t big_ncand;        // IFs with more candidates use the multi-kernel select (0: never)
  uint32_t* big_list;        // [n] IFs on the multi-kernel select path, [n] = their count
  uint32_t inject;           // test-only fault injection (SIF_TEST_INJECT): bit 0 = sampled bracket misses
};

// Rebind IF i of an uploaded plan (sif_enc_set_input): input, payload buffer, seed.
__global__ void set_enc_input_kernel(IfInfo* info, const void* x, uint8_t* out, uint64_t seed) {
  info->x = x;
  info->out = out;
  info->seed = seed;
}

__device__ __forceinline__ void prof_mark(const EArgs& a, int ifi, int k) {
  if (a.prof && threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.prof[(uint64_t)ifi * 32 + k] = t;
  }
}

// candidate list of an IF: (float bits, flat index) entries
__device__ __forceinline__ uint2* le(const EArgs& a, const IfInfo& f) {
  return reinterpret_cast<uint2*>(a.ws + f.list_off);
}
// K3 gather spill, then the regrouped members (K4 output): per chunk a slot of CH entries
__device__ __forceinline__ uint2* me(const EArgs& a, const IfInfo& f) {
  return reinterpret_cast<uint2*>(a.ws + f.gat_off);
}

// quant.py:59-62 in float64: floor((v - vmin)/o64 + 0.5) clipped to [0, levels].  The
// reciprocal fast path is exact except within 1e-6 of a rounding boundary, where the
// correctly rounded float64 division is used.
__device__ __forceinline__ uint32_t quant_code(uint32_t key, double vmin64, double o64, double inv64,
                                               uint32_t levels) {
  const double v = (double)__uint_as_float(key);
  const double dl = __dsub_rn(v, vmin64);
  double t = __dadd_rn(__dmul_rn(dl, inv64), 0.5);
  double f = floor(t);
  const double fr = __dsub_rn(t, f);
  if (fr < 1e-6 || fr > 0.999999) {
    t = __dadd_rn(__ddiv_rn(dl, o64), 0.5);
    f = floor(t);
  }
  if (!(f > 0.0)) return 0u;
  return f >= (double)levels ? levels : (uint32_t)f;
}


// ---------------------------------------------------------------------------------------
// List of (float bits, flat index) pairs: SMEM up to `cap` entries, global beyond.
struct List {
  uint2* s;
  uint2* g;
  uint32_t cap;
  __device__ __forceinline__ void set(uint32_t i, uint32_t b, uint32_t x) const {
    if (i < cap) s[i] = make_uint2(b, x);
    else __stcg(g + (i - cap), make_uint2(b, x));
  }
  __device__ __forceinline__ uint2 get(uint32_t i) const { return i < cap ? s[i] : __ldcg(g + (i - cap)); }
};

// Visit every list element (order-free) as f(bits, idx, true).  Global parts are read U
// entries per thread per step with independent 8-byte loads (U loads in flight).
template <int NT, int U = 4, class F>
__device__ __forceinline__ void list_foreach(const List& L, uint32_t n, F f) {
  const uint32_t ns = n < L.cap ? n : L.cap;
  for (uint32_t i = threadIdx.x; i < ns; i += NT) {
    const uint2 e = L.s[i];
    f(e.x, e.y, true);
  }
  if (n > L.cap) {
    const uint32_t m = n - L.cap;
    for (uint32_t i0 = 0; i0 < m; i0 += U * NT) {
      uint2 e[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const uint32_t i = i0 + threadIdx.x + k * NT;
        e[k] = i < m ? __ldcg(L.g + i) : make_uint2(0, 0);
      }
#pragma unroll
      for (int k = 0; k < U; ++k)
        if (i0 + threadIdx.x + k * NT < m) f(e[k].x, e[k].y, true);
    }
  }
}

struct GatE {
  uint32_t key;
  uint32_t idx;
  uint64_t sec;
};

struct SelSh {
  uint64_t scan[40];
  uint32_t red[72];  // >= 2 * (NT / 32) + 1 for NT <= 1024
  uint32_t fd_digit;
  uint64_t fd_above, fd_eq;
  uint32_t fd_found;
  uint32_t gcount;
  uint32_t sel_key;
  uint64_t sel_sec;
  uint32_t sel_found;
  uint32_t cnt[8];
};

// Find digit d of histogram H (nb bins) with above(d) < r <= above(d) + H[d], from the top.
template <int NT>
__device__ void find_digit(SelSh& sh, const uint32_t* H, int nb, uint64_t r) {
  const int per = (nb + NT - 1) / NT;
  uint64_t s = 0;
  for (int k = 0; k < per; ++k) {
    const int b = nb - 1 - (threadIdx.x * per + k);
    if (b >= 0) s += H[b];
  }
  uint64_t tot;
  const uint64_t ex = block_excl_scan_u64(s, sh.scan, &tot);
  if (threadIdx.x == 0) sh.fd_found = 0;
  __syncthreads();
  if (ex < r && r <= ex + s) {
    uint64_t cum = ex;
    for (int k = 0; k < per; ++k) {
      const int b = nb - 1 - (threadIdx.x * per + k);
      if (b < 0) break;
      const uint64_t h = H[b];
      if (cum < r && r <= cum + h) {
        sh.fd_digit = (uint32_t)b;
        sh.fd_above = cum;
        sh.fd_eq = h;
        sh.fd_found = 1;
        break;
      }
      cum += h;
    }
  }
  __syncthreads();
}

// Multi-level radix select ("r-th largest") on keys of `nbits` bits (64 or <= 33) over list
// elements accepted by fn(bits, idx, &key); keys must be distinct (splitmix64 hashes and
// flat indices are).  As soon as the bin holding rank r has <= GCAP elements they are
// gathered and ranked directly.  Used for huge single-value tie sets.
struct GatE;
template <int NT, int U = 4, class KeyFn>
__device__ uint64_t radix_select64(SelSh& sh, uint32_t* hist, const List& L, uint32_t n, uint64_t r, KeyFn fn,
                                   int nbits = 64);

template <int NT, int U, class KeyFn>
__device__ uint64_t radix_select64(SelSh& sh, uint32_t* hist, const List& L, uint32_t n, uint64_t r, KeyFn fn,
                                   int nbits) {
  GatE* gl = reinterpret_cast<GatE*>(hist + 2 * HB);
  uint64_t prefix = 0, mask = 0;
  for (int hi = nbits; hi > 0;) {
    const int wdt = hi >= 11 ? 11 : hi;
    const int shf = hi - wdt, nb = 1 << wdt;
    for (int i = threadIdx.x; i < nb; i += NT) hist[i] = 0;
    __syncthreads();
    list_foreach<NT, U>(L, n, [&](uint32_t b, uint32_t x, bool v) {
      uint64_t k = 0;
      if (v && fn(b, x, k) && (k & mask) == prefix) atomicAdd(&hist[(int)((k >> shf) & (uint64_t)(nb - 1))], 1u);
    });
    __syncthreads();
    find_digit<NT>(sh, hist, nb, r);
    prefix |= (uint64_t)sh.fd_digit << shf;
    mask |= (uint64_t)(nb - 1) << shf;
    r -= sh.fd_above;
    const uint64_t cnt = sh.fd_eq;
    __syncthreads();
    hi = shf;
    if (hi > 0 && cnt <= GCAP) {
      // small bin: gather its keys and take the r-th largest directly
      if (threadIdx.x == 0) sh.gcount = 0;
      __syncthreads();
      list_foreach<NT, U>(L, n, [&](uint32_t b, uint32_t x, bool v) {
        uint64_t k = 0;
        if (v && fn(b, x, k) && (k & mask) == prefix) gl[atomicAdd(&sh.gcount, 1u)].sec = k;
      });
      __syncthreads();
      const uint32_t m = sh.gcount;
      for (uint32_t i = threadIdx.x; i < m; i += NT) {
        const uint64_t ki = gl[i].sec;
        uint32_t rank = 0;
        for (uint32_t j = 0; j < m; ++j) rank += gl[j].sec > ki;
        if (rank == r - 1) sh.sel_sec = ki;
      }
      __syncthreads();
      const uint64_t res = sh.sel_sec;
      __syncthreads();
      return res;
    }
  }
  return prefix;
}

// Result of an exact select: the element at 1-based rank r by (key desc, sec asc).
struct SelRes {
  uint32_t key;
  uint64_t sec;
  uint64_t n_gt, n_eq, r_eq;
  int all_ties;
};

// Exact select over the list elements accepted by pred, ordered by (keyf desc, secf asc),
// restricted to keys in [klo, khi).  Levels of <= 2048-bin histograms narrow the range to
// the bin holding rank r; the bin's elements are gathered and ranked exactly.  A bin that
// is one key value with more than GCAP members resolves the secondary order by a radix
// select on the secondary key.  scratch: 2*HB u32 + GCAP GatE.
template <int NT, int U = 4, class Pred, class KeyF, class SecF>
__device__ SelRes select_exact(SelSh& sh, uint32_t* scratch, const List& L, uint32_t n, Pred pred, KeyF keyf,
                               SecF secf, uint64_t klo, uint64_t khi, uint64_t r, int sec_bits = 64) {
  constexpr int NW = NT / 32;
  uint32_t* hist = scratch;
  GatE* gl = reinterpret_cast<GatE*>(scratch + 2 * HB);
  const int tid = threadIdx.x;
  uint64_t n_gt = 0, cnt = 0;
  for (;;) {
    const uint64_t span = khi - klo;
    const int bl = span > 1 ? 64 - __clzll(span - 1) : 0;
    const int shf = bl > 11 ? bl - 11 : 0;
    const int nb = (int)(((span - 1) >> shf) + 1);
    for (int i = tid; i < nb; i += NT) hist[i] = 0;
    __syncthreads();
    list_foreach<NT, U>(L, n, [&](uint32_t b, uint32_t x, bool v) {
      if (v && pred(b, x)) {
        const uint64_t k = keyf(b);
        if (k >= klo && k < khi) atomicAdd(&hist[(int)((k - klo) >> shf)], 1u);
      }
    });
    __syncthreads();
    find_digit<NT>(sh, hist, nb, r);
    const uint64_t dg = sh.fd_digit;
    n_gt += sh.fd_above;
    r -= sh.fd_above;
    cnt = sh.fd_eq;
    klo = klo + (dg << shf);
    const uint64_t nhi = klo + (1ull << shf);
    khi = nhi < khi ? nhi : khi;
    __syncthreads();
    if (cnt <= GCAP || shf == 0) break;
  }
  SelRes res;
  if (cnt > GCAP) {
    res.key = (uint32_t)klo;
    res.n_gt = n_gt;
    res.n_eq = cnt;
    res.r_eq = r;
    res.all_ties = r == cnt;
    // the secondary key of the r-th tie is needed even when r == cnt (every tie selected):
    // MS cuts (msplit.py:64) place the block boundary at that element's flat index
    const uint32_t kk = (uint32_t)klo;
    // smallest secondary keys first: select the r-th largest of (2^sec_bits - 1 - sec)
    const uint64_t smax = sec_bits >= 64 ? ~0ull : ((1ull << sec_bits) - 1ull);
    const uint64_t top = radix_select64<NT, U>(sh, hist, L, n, r, [&](uint32_t b, uint32_t x, uint64_t& k) {
      if (!pred(b, x) || keyf(b) != kk) return false;
      k = smax - secf(b, x);
      return true;
    }, sec_bits);
    res.sec = smax - top;
    return res;
  }
  if (tid == 0) sh.gcount = 0;
  __syncthreads();
  list_foreach<NT, U>(L, n, [&](uint32_t b, uint32_t x, bool v) {
    bool in = v && pred(b, x);
    const uint64_t k = in ? keyf(b) : 0;
    in = in && k >= klo && k < khi;
    if (in) {
      const uint32_t p = atomicAdd(&sh.gcount, 1u);
      gl[p].key = (uint32_t)k;
      gl[p].idx = x;
      gl[p].sec = secf(b, x);
    }
  });
  __syncthreads();
  const uint32_t m = (uint32_t)cnt;
  if (tid == 0) sh.sel_found = 0;
  __syncthreads();
  if (m <= 256) {
    for (uint32_t i = tid; i < m; i += NT) {
      const uint32_t ki = gl[i].key;
      const uint64_t si = gl[i].sec;
      uint32_t rank = 0;
      for (uint32_t j = 0; j < m; ++j) {
        const uint32_t kj = gl[j].key;
        rank += (kj > ki) || (kj == ki && gl[j].sec < si);
      }
      if (rank == r - 1) {
        sh.sel_key = ki;
        sh.sel_sec = si;
        sh.sel_found = 1;
      }
    }
  } else {
    uint32_t p2 = 1;
    while (p2 < m) p2 <<= 1;
    for (uint32_t i = m + tid; i < p2; i += NT) { gl[i].key = 0; gl[i].sec = ~0ull; gl[i].idx = 0; }
    __syncthreads();
    for (uint32_t k = 2; k <= p2; k <<= 1) {
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        for (uint32_t i = tid; i < p2; i += NT) {
          const uint32_t ixj = i ^ j;
          if (ixj > i) {
            const GatE A = gl[i], Bv = gl[ixj];
            const bool a_first = A.key > Bv.key || (A.key == Bv.key && A.sec < Bv.sec);
            const bool up = (i & k) == 0;
            if (up != a_first) { gl[i] = Bv; gl[ixj] = A; }
          }
        }
        __syncthreads();
      }
    }
    if (tid == 0) {
      sh.sel_key = gl[r - 1].key;
      sh.sel_sec = gl[r - 1].sec;
      sh.sel_found = 1;
    }
  }
  __syncthreads();
  const uint32_t ks = sh.sel_key;
  uint32_t gt = 0, eq = 0;
  for (uint32_t i = tid; i < m; i += NT) {
    gt += gl[i].key > ks;
    eq += gl[i].key == ks;
  }
  gt = __reduce_add_sync(0xFFFFFFFFu, gt);
  eq = __reduce_add_sync(0xFFFFFFFFu, eq);
  if ((tid & 31) == 0) { sh.red[tid >> 5] = gt; sh.red[NW + (tid >> 5)] = eq; }
  __syncthreads();
  uint64_t tgt = 0, teq = 0;
  for (int w = 0; w < NW; ++w) { tgt += sh.red[w]; teq += sh.red[NW + w]; }
  res.key = ks;
  res.sec = sh.sel_sec;
  res.n_gt = n_gt + tgt;
  res.n_eq = teq;
  res.r_eq = r - tgt;
  res.all_ties = res.r_eq == teq;
  __syncthreads();
  return res;
}

// ---------------------------------------------------------------------------------------
// A unit is UE = 512 consecutive elements of a chunk, streamed by one warp; lane l owns the
// 16 contiguous elements [16l, 16l+16) (fp32: four 128-bit loads, bf16: two).
struct Raw {
  uint4 r[4];
};

__device__ __forceinline__ void load_unit(const void* xp, uint32_t dtype, uint32_t e0, uint32_t n, Raw& raw) {
  const int lane = threadIdx.x & 31;
  const uint32_t b = 16u * lane;
  if (dtype == SIF_DTYPE_F32) {
    const uint32_t* x = reinterpret_cast<const uint32_t*>(xp) + e0 + b;
    if (b + 16 <= n) {
#pragma unroll
      for (int j = 0; j < 4; ++j) raw.r[j] = __ldcs(reinterpret_cast<const uint4*>(x) + j);  // read once: evict-first
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t c[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) c[k] = b + 4 * j + k < n ? __ldg(x + 4 * j + k) : 0u;
        raw.r[j] = make_uint4(c[0], c[1], c[2], c[3]);
      }
    }
  } else {
    const unsigned short* x = reinterpret_cast<const unsigned short*>(xp) + e0 + b;
    raw.r[2] = make_uint4(0, 0, 0, 0);
    raw.r[3] = make_uint4(0, 0, 0, 0);
    if (b + 16 <= n) {
#pragma unroll
      for (int j = 0; j < 2; ++j) raw.r[j] = __ldcs(reinterpret_cast<const uint4*>(x) + j);  // read once: evict-first
    } else {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        uint32_t c[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t e = b + 8 * j + 2 * k;
          const uint32_t lo16 = e < n ? (uint32_t)__ldg(x + 8 * j + 2 * k) : 0u;
          const uint32_t hi16 = e + 1 < n ? (uint32_t)__ldg(x + 8 * j + 2 * k + 1) : 0u;
          c[k] = lo16 | (hi16 << 16);
        }
        raw.r[j] = make_uint4(c[0], c[1], c[2], c[3]);
      }
    }
  }
}

__device__ __forceinline__ uint32_t u4c(const uint4& q, int k) {
  return k == 0 ? q.x : k == 1 ? q.y : k == 2 ? q.z : q.w;
}

// Classify one unit (n valid elements from flat index e0): candidates (|x| >= lo for x >= 0,
// |x| >= lo_neg for x < 0) are written in flat order to the warp staging `stage` as
// (bits, flat index); returns the count (warp-uniform).  asym: lo != lo_neg, then `clo`
// accumulates the count of |x| >= lo (otherwise that count is the candidate count).
template <int DT>
__device__ __forceinline__ uint32_t classify_unit(const Raw& raw, uint32_t e0, uint32_t n, uint32_t lo, uint32_t lo_neg,
                                                  bool asym, uint2* stage, uint32_t& clo) {
  const int lane = threadIdx.x & 31;
  const uint32_t b0 = 16u * lane;
  uint32_t v[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    if (DT == SIF_DTYPE_F32) v[k] = u4c(raw.r[k >> 2], k & 3);
    else {
      const uint32_t wv = u4c(raw.r[k >> 3], (k >> 1) & 3);
      v[k] = (k & 1) ? (wv & 0xFFFF0000u) : (wv << 16);
    }
  }
  const uint32_t nl = n >= b0 + 16 ? 16u : (n > b0 ? n - b0 : 0u);
  const uint32_t vmask = nl == 16 ? 0xFFFFu : ((1u << nl) - 1u);
  uint32_t m = 0;
  if (!asym) {
#pragma unroll
    for (int k = 0; k < 16; ++k) m |= ((v[k] & 0x7FFFFFFFu) >= lo ? 1u : 0u) << k;
  } else {
    uint32_t ml = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const uint32_t key = v[k] & 0x7FFFFFFFu;
      m |= (key >= ((v[k] >> 31) ? lo_neg : lo) ? 1u : 0u) << k;
      ml |= (key >= lo ? 1u : 0u) << k;
    }
    clo += __popc(ml & vmask);
  }
  m &= vmask;
  const uint32_t cnt = __popc(m);
  const uint32_t incl = warp_incl_scan_u32(cnt);
  uint32_t pos = incl - cnt;
  const uint32_t ex = e0 + b0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const bool p = (m >> k) & 1u;
    if (p) stage[pos] = make_uint2(v[k], ex + k);
    pos += p ? 1u : 0u;
  }
  return __shfl_sync(0xFFFFFFFFu, incl, 31);
}

__device__ __forceinline__ uint32_t classify_any(uint32_t dtype, const Raw& raw, uint32_t e0, uint32_t n, uint32_t lo,
                                                 uint32_t lo_neg, bool asym, uint2* stage, uint32_t& clo) {
  if (dtype == SIF_DTYPE_BF16) return classify_unit<SIF_DTYPE_BF16>(raw, e0, n, lo, lo_neg, asym, stage, clo);
  return classify_unit<SIF_DTYPE_F32>(raw, e0, n, lo, lo_neg, asym, stage, clo);
}

// Copy a staged unit (cnt candidates) to the IF's list at `dst`; max key, digit histogram
// (if hist) and digit range of the candidates.
__device__ __forceinline__ void emit_unit(const uint2* stage, uint32_t cnt, uint2* dst, uint32_t* hist, uint32_t& mk,
                                          uint32_t& dmin, uint32_t& dmax) {
  const int lane = threadIdx.x & 31;
  for (uint32_t k = lane; k < cnt; k += 32) {
    const uint2 e = stage[k];
    dst[k] = e;
    const uint32_t key = e.x & 0x7FFFFFFFu;
    mk = max(mk, key);
    if (hist) {
      const uint32_t d = key >> DSH;
      atomicAdd(&hist[((e.x >> 31) ? ND : 0) + d], 1u);
      dmin = min(dmin, d);
      dmax = max(dmax, d);
    }
  }
}

// Unit geometry: flat start and valid count of unit (c, u).
__device__ __forceinline__ void unit_span(const EArgs& a, const IfInfo& f, uint32_t c, uint32_t u, uint32_t& e0,
                                          uint32_t& n) {
  e0 = a.ch_e0[c] + u * (uint32_t)UE;
  n = e0 < f.T ? (uint32_t)min((uint64_t)UE, f.T - e0) : 0u;
}

// ---------------------------------------------------------------------------------------
// K1: per-IF setup: accumulators and the sampled bracket lo (speculation only: a missed
// bracket is detected in K3 and the IF re-streamed).
// SMALL: a batch whose IFs all fit one chunk (<= 4096 elements): narrow CTAs and only the
// exact-tau path, so many IFs share an SM.
// Candidate bracket lo for IF f (K1): the exact tau key for IFs of <= EXACT_T elements (3
// radix levels in shared memory), otherwise a sampled lower bound (4096 elements, 13-bit
// key histogram, 3-sigma margin); 1 when no bracket applies.  sh8k: >= EXACT_T + 2048 u32
// of shared memory (8192 + 2048 covers both).
template <int NT, bool SMALL>
__device__ __forceinline__ uint32_t bracket_lo(const EArgs& a, const IfInfo& f, uint32_t* sh8k, SelSh& sh) {
  constexpr int EXACT_T = SMALL ? CH : 8192;  // IFs up to this size get the exact tau key as lo
  const int tid = threadIdx.x;
  const uint64_t T = f.T, kk = f.kk;
  uint32_t lo = 1;
  if (T <= EXACT_T && kk > 0) {
    // exact: the kk-th largest |x| key by a 3-level radix select in shared memory
    uint32_t* keys = sh8k;
    uint32_t* h = sh8k + (SMALL ? CH : 8192);
    const uint32_t n = (uint32_t)T;
    uint32_t kor = 0, kand = 0xFFFFFFFFu;
    for (uint32_t e = tid; e < n; e += NT) {
      const uint32_t b = f.dtype == SIF_DTYPE_F32 ? __ldg(reinterpret_cast<const uint32_t*>(f.x) + e)
                                                  : (uint32_t)__ldg(reinterpret_cast<const unsigned short*>(f.x) + e) << 16;
      keys[e] = b & 0x7FFFFFFFu;
      kor |= b & 0x7FFFFFFFu;
      kand &= b & 0x7FFFFFFFu;
    }
    // bits equal in every key (e.g. the low 16 bits of bf16 data) need no histogram level
    kor = __reduce_or_sync(0xFFFFFFFFu, kor);
    kand = __reduce_and_sync(0xFFFFFFFFu, kand);
    if ((tid & 31) == 0) { sh.red[tid >> 5] = kor; sh.red[NT / 32 + (tid >> 5)] = kand; }
    __syncthreads();
    uint32_t vary = 0, cand = 0xFFFFFFFFu;
    for (int w = 0; w < NT / 32; ++w) { vary |= sh.red[w]; cand &= sh.red[NT / 32 + w]; }
    vary ^= cand;  // bits that differ between some keys
    uint64_t r = kk;
    uint32_t prefix = 0, mask = 0;
    const int shifts[3] = {20, 9, 0}, widths[3] = {11, 11, 9};
    for (int lev = 0; lev < 3; ++lev) {
      const int shf = shifts[lev], nb = 1 << widths[lev];
      const uint32_t lmask = (uint32_t)(nb - 1) << shf;
      if ((vary & lmask) == 0) {  // one bin holds every remaining key: its digit is the common bits
        prefix |= cand & lmask;
        mask |= lmask;
        continue;
      }
      for (int k = tid; k < nb; k += NT) h[k] = 0;
      __syncthreads();
      for (uint32_t e = tid; e < n; e += NT) {
        const uint32_t key = keys[e];
        if ((key & mask) == prefix) atomicAdd(&h[(key >> shf) & (uint32_t)(nb - 1)], 1u);
      }
      __syncthreads();
      find_digit<NT>(sh, h, nb, r);
      prefix |= sh.fd_digit << shf;
      mask |= lmask;
      r -= sh.fd_above;
      __syncthreads();
    }
    lo = prefix > 0 ? prefix : 1u;  // tau == 0: every nonzero is a candidate
  } else if (!SMALL && T > 32768 && kk > 0 && 2 * kk <= T) {
    constexpr int NSECT = 512, SB = 8192, PERT = NSECT / NT;
    for (int k = tid; k < SB; k += NT) sh8k[k] = 0;
    uint32_t sv[PERT][8];
#pragma unroll
    for (int k = 0; k < PERT; ++k) {
      const int j = tid + k * NT;
      // low-discrepancy (Weyl) sector positions avoid aliasing with row structure
      const uint64_t nsec = T / 8;
      const uint64_t frac = (uint64_t)(uint32_t)((uint32_t)j * 0x9E3779B9u);
      const uint64_t e = ((frac * nsec) >> 32) * 8;
      if (f.dtype == SIF_DTYPE_F32) {
        const uint4* q4 = reinterpret_cast<const uint4*>(reinterpret_cast<const uint32_t*>(f.x) + e);
        const uint4 v0 = __ldg(q4), v1 = __ldg(q4 + 1);
        sv[k][0] = v0.x; sv[k][1] = v0.y; sv[k][2] = v0.z; sv[k][3] = v0.w;
        sv[k][4] = v1.x; sv[k][5] = v1.y; sv[k][6] = v1.z; sv[k][7] = v1.w;
      } else {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const unsigned short*>(f.x) + e));
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) { sv[k][2 * q] = w[q] << 16; sv[k][2 * q + 1] = w[q] & 0xFFFF0000u; }
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < PERT; ++k)
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t key = sv[k][q] & 0x7FFFFFFFu;
        if (key && key < kNonFiniteKey) atomicAdd(&sh8k[key >> 18], 1u);
      }
    __syncthreads();
    const double S = NSECT * 8.0;
    const double qf = (double)kk / (double)T;
    const double sd = sqrt(qf * (1.0 - qf) * S);
    const double rlo = ceil(qf * S + 3.0 * sd + 2.0);
    find_digit<NT>(sh, sh8k, SB, (uint64_t)rlo);
    lo = sh.fd_found ? (sh.fd_digit << 18) : 1u;
    if (lo == 0) lo = 1;
    if (a.inject & 1u) lo = 0x7F000000u;  // fault injection (tests): the bracket misses, K3 re-streams
  }
  return lo;
}

template <int NT, bool SMALL>
__global__ void __launch_bounds__(NT) enc_prep(EArgs a) {
  __shared__ uint32_t sh8k[(SMALL ? CH : 8192) + 2048];
  __shared__ SelSh sh;
  const int i = blockIdx.x, tid = threadIdx.x;
  const IfInfo f = a.info[i];
  IfSt& st = a.st[i];
  if (i == 0 && tid == 0) a.big_list[a.n] = 0;
  if (f.path == PATH_TOKEN) return;  // encoded by enc_token
  for (int b = tid; b < a.maxb; b += NT) { st.bmin[b] = 0x7FFFFFFFu; st.bmax[b] = 0u; }
  for (int k = tid; k < a.maxb * 16; k += NT) st.S[k] = 0ull;
  for (int b = tid; b < a.maxb; b += NT) st.bcount[b] = 0u;
  // (the IF's digit histogram is zeroed by enc_select after it has read it, and by
  //  sif_enc_upload before the first run)
  uint32_t lo = bracket_lo<NT, SMALL>(a, f, sh8k, sh);
  uint32_t lo_neg = lo;
  if (a.lam > 0.0 && lo > 1) {
    const double t = __dmul_rn(__dsub_rn(1.0, a.lam), (double)__uint_as_float(lo));
    const uint32_t k2 = __float_as_uint(__double2float_rd(t));
    lo_neg = k2 > 1 ? k2 : 1u;
  }
  if (tid == 0) {
    st.lo = lo; st.lo_neg = lo_neg; st.ncand = 0; st.maxkey = 0; st.cnt_lo = 0; st.err = E_NONE; st.flags = 0;
    st.P = 0; st.crc_acc = 0; st.seg_done = 0; st.sel_phase = 0;
  }
}

// ---------------------------------------------------------------------------------------
// K2: stream chunks.  Each CTA owns a contiguous range of chunks; warp w streams unit w of
// every chunk (UE elements, 128-bit loads, two units prefetched), stages its candidates in
// flat order, reserves list space with one atomic per unit and copies them out coalesced.
// Per-IF reductions (max key, count >= lo, SMEM digit histogram) are flushed when the IF
// changes, so the hot loop has no CTA barrier.
__device__ __forceinline__ void flush_if_stream(const EArgs& a, uint32_t ifi, uint32_t* hist, uint32_t& mk,
                                                uint32_t& clo, uint32_t& dmin, uint32_t& dmax, uint32_t* sdr) {
  const int tid = threadIdx.x, lane = tid & 31;
  IfSt& st = a.st[ifi];
  mk = __reduce_max_sync(0xFFFFFFFFu, mk);
  clo = __reduce_add_sync(0xFFFFFFFFu, clo);
  const uint32_t d0 = __reduce_min_sync(0xFFFFFFFFu, dmin), d1 = __reduce_max_sync(0xFFFFFFFFu, dmax);
  if (lane == 0) {
    atomicMax(&st.maxkey, mk);
    if (clo) atomicAdd(&st.cnt_lo, clo);
    atomicMin(&sdr[0], d0);
    atomicMax(&sdr[1], d1);
  }
  __syncthreads();
  const int hs = a.info[ifi].hslot;
  if (hs >= 0 && sdr[0] <= sdr[1]) {
    uint32_t* gh = a.hist + (uint64_t)hs * 2 * ND;
    const uint32_t lo = sdr[0], nr = sdr[1] - sdr[0] + 1;
    for (uint32_t k = tid; k < 2 * nr; k += CNT) {
      const uint32_t d = (k < nr ? 0u : (uint32_t)ND) + lo + (k < nr ? k : k - nr);
      const uint32_t h = hist[d];
      if (h) { atomicAdd(gh + d, h); hist[d] = 0; }
    }
  }
  __syncthreads();
  if (tid == 0) { sdr[0] = 0xFFFFFFFFu; sdr[1] = 0; }
  mk = 0; clo = 0; dmin = 0xFFFFFFFFu; dmax = 0;
  __syncthreads();
}

__global__ void __launch_bounds__(CNT, 3) enc_stream(EArgs a) {
  extern __shared__ __align__(16) uint8_t dsm_raw[];
  uint32_t* dsm = reinterpret_cast<uint32_t*>(dsm_raw);
  __shared__ uint32_t sdr[2];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  uint2* stage = reinterpret_cast<uint2*>(dsm) + w * UE;
  uint32_t* hist = dsm + (CNT / 32) * 2 * UE;
  for (int k = tid; k < 2 * ND; k += CNT) hist[k] = 0;
  if (tid == 0) { sdr[0] = 0xFFFFFFFFu; sdr[1] = 0; }
  __syncthreads();
  const uint32_t nch = (uint32_t)a.nch;
  const uint32_t c0 = (uint32_t)((uint64_t)nch * blockIdx.x / gridDim.x);
  const uint32_t c1 = (uint32_t)((uint64_t)nch * (blockIdx.x + 1) / gridDim.x);
  if (c0 >= c1) return;
  uint32_t cur = a.ch_if[c0];
  IfInfo f = a.info[cur];
  uint32_t lo = a.st[cur].lo, lo_neg = a.st[cur].lo_neg;
  uint32_t mk = 0, clo = 0, dmin = 0xFFFFFFFFu, dmax = 0;
  Raw r0, r1;
  auto prefetch = [&](uint32_t c, Raw& r) {
    const IfInfo& g = a.info[a.ch_if[c]];
    uint32_t e0, n;
    unit_span(a, g, c, (uint32_t)w, e0, n);
    if (n) load_unit(g.x, g.dtype, e0, n, r);
  };
  prefetch(c0, r0);
  if (c0 + 1 < c1) prefetch(c0 + 1, r1);
  for (uint32_t c = c0; c < c1; ++c) {
    const uint32_t ifi = a.ch_if[c];
    if (ifi != cur) {
      flush_if_stream(a, cur, hist, mk, clo, dmin, dmax, sdr);
      cur = ifi;
      f = a.info[ifi];
      lo = a.st[ifi].lo;
      lo_neg = a.st[ifi].lo_neg;
    }
    Raw r2;
    if (c + 2 < c1) prefetch(c + 2, r2);
    uint32_t e0, n;
    unit_span(a, f, c, (uint32_t)w, e0, n);
    const bool asym = lo != lo_neg;
    uint32_t cnt = 0;
    if (n) cnt = classify_any(f.dtype, r0, e0, n, lo, lo_neg, asym, stage, clo);
    if (!asym && lane == 0) clo += cnt;
    uint32_t off = 0;
    if (lane == 0) {
      off = cnt ? atomicAdd(&a.st[ifi].ncand, cnt) : 0u;
      a.u_off[(uint64_t)c * UNITS + w] = off;
      a.u_cnt[(uint64_t)c * UNITS + w] = cnt;
    }
    off = __shfl_sync(0xFFFFFFFFu, off, 0);
    __syncwarp();
    emit_unit(stage, cnt, le(a, f) + off, f.hslot >= 0 ? hist : nullptr, mk, dmin, dmax);
    __syncwarp();
    r0 = r1;
    r1 = r2;
  }
  flush_if_stream(a, cur, hist, mk, clo, dmin, dmax, sdr);
}

// The IF's digit histogram is dead once enc_select has read it: zero it for the next run
// (plain stores at the end of the kernel, so nothing waits on them).
__device__ __forceinline__ void zero_hist(const EArgs& a, const IfInfo& f) {
  if (f.hslot < 0) return;
  uint4* gh = reinterpret_cast<uint4*>(a.hist + (uint64_t)f.hslot * 2 * ND);
  for (int k = threadIdx.x; k < 2 * ND / 4; k += blockDim.x) gh[k] = make_uint4(0, 0, 0, 0);
}

// ---------------------------------------------------------------------------------------
// K3: per-IF selection.
struct K3Sh {
  SelSh s;
  uint32_t cursor;
  uint32_t nA, nB;
  uint32_t keptA[2];
  uint32_t fullb[2], lowd[2];  // lambda > 0: per sign the digit of the smallest kept key, its bin size
  uint64_t cnt_nz;
  uint32_t pend_n;
  uint32_t pend_s[MAXB], pend_d[MAXB], pend_r[MAXB], pend_ci[MAXB], pend_reg[MAXB];
  uint32_t reg_off[MAXB], reg_cnt[MAXB];
};

// Three launches: PH 0 resolves everything for the uncommon paths (lambda > 0, tau == 0,
// k == 0, tiny plane counts) and, on the common path, only the digit of tau; the tau bin is
// then gathered by all SMs (enc_gather<1>), PH 1 selects tau inside it, counts the kept
// elements, finds every MS cut's digit and resolves the cuts inside tau's bin; the other
// cut bins are gathered by all SMs (enc_gather<2>) and PH 2 resolves those cuts.
// The body of K3 for IF `ifi`, run by every thread of a CTA of NT threads.  dsm: dynamic
// shared memory of kSmemSelect bytes (hist | scratch | gbuf).  FUSED: called by the fused
// per-IF encoder (enc_fused), whose stream phase already left the IF's digit histogram in
// `hist` and resolved any bracket miss; no multi-kernel split.
template <int PH, int NT, bool FUSED, bool DEEP = false, bool NOCLS = false>
__device__ __forceinline__ void select_if(const EArgs& a, const int ifi, uint32_t* dsm, K3Sh& k3,
                                          const List* Lin = nullptr) {
  // loads in flight per thread in list passes: deep for the big-IF phases and for a batch
  // with lambda > 0 IFs large enough that their whole select runs here (DEEP)
  constexpr int LU = (PH > 0 || DEEP) ? 16 : 8;
  SelSh& sh = k3.s;
  uint32_t* hist = dsm;                         // 2*ND
  uint32_t* scratch = dsm + 2 * ND;             // 2*HB + GCAP*4
  uint32_t* gbuf = scratch + 2 * HB + GCAP * 4; // 2*GSM (also the re-stream stage)
  const int tid = threadIdx.x;
  const IfInfo f = a.info[ifi];
  IfSt& st = a.st[ifi];
  const uint64_t kk = f.kk, seed = f.seed;
  if (PH == 0 && st.sel_phase == 4) return;  // resolved by enc_select_tiny
  if (PH > 0) {
    if (st.sel_phase != (uint32_t)PH && !(PH == 2 && st.sel_phase == 5u)) return;
    if (PH == 2) {
      // cut bins gathered into their regions of the gather area: exact selects, one CTA
      // per pending cut (blockIdx.y); sel_phase stays 2 until the next run's enc_prep
      auto key31 = [](uint32_t b) -> uint64_t { return b & 0x7FFFFFFFu; };
      const uint32_t np = st.pend_n;
      uint2* gat = me(a, f);
      // lambda > 0: the partial bin at the kept threshold was gathered whole; members are the
      // kept candidates (KeptCtx::kept over the IfSt written by enc_select<0>)
      const uint32_t flg = st.flags;
      const uint64_t cks = st.ck_star, hst = st.h_star;
      const double tp = st.tau_p, tm = st.tau_m;
      auto kept = [=](uint32_t b, uint32_t x) -> bool {
        if (!(flg & F_USE_CLS)) return true;
        uint64_t c = b & 0x7FFFFFFFu;
        const double v = (double)__uint_as_float(b);
        if (v > tp || v < tm) c |= 1ull << 31;
        if (c != cks) return c > cks;
        return (flg & F_TIE_ALL) || splitmix(seed, x) <= hst;
      };
      for (uint32_t p = blockIdx.y; p < np; p += gridDim.y) {
        const uint32_t g = st.pend_reg[p];
        const List Bp{nullptr, gat + st.reg_off[g], 0};
        const uint32_t dc = st.pend_d[p];
        const SelRes r = select_exact<NT, LU>(
            sh, scratch, Bp, st.reg_cnt[g], kept, key31,
            [](uint32_t, uint32_t x) -> uint64_t { return x; }, (uint64_t)dc << DSH, (uint64_t)(dc + 1) << DSH,
            st.pend_r[p], 31);
        if (tid == 0) { st.cut_key[st.pend_ci[p]] = r.key; st.cut_idx[st.pend_ci[p]] = (uint32_t)r.sec; }
        __syncthreads();
      }
      return;
    }
  }
  if (PH == 0 && st.maxkey >= kNonFiniteKey) {
    if (f.hslot >= 0) {
      uint4* gh = reinterpret_cast<uint4*>(a.hist + (uint64_t)f.hslot * 2 * ND);
      for (int k = tid; k < 2 * ND / 4; k += NT) gh[k] = make_uint4(0, 0, 0, 0);
    }
    if (tid == 0) {
      st.err = E_NONFINITE;
      if (a.atkf_only) a.status[ifi] = SIF_ERR_NONFINITE;
    }
    return;
  }
  uint32_t lo = PH == 0 ? st.lo : st.sel_lo, lo_neg = st.lo_neg;
  const uint32_t floor_lo = a.atkf_only ? 0u : 1u;
  uint32_t ncand = st.ncand;
  bool hist_ok = false;
  prof_mark(a, ifi, 0);
  if (FUSED) {
    hist_ok = true;
  } else if (PH == 0 && kk > 0 && st.cnt_lo < kk && lo > floor_lo) {
    // bracket missed (or tau == 0): re-stream keeping every nonzero (every element in
    // ATKF-only mode); this CTA writes the list in chunk order and the histogram in SMEM
    lo = floor_lo;
    lo_neg = floor_lo;
    for (int k = tid; k < 2 * ND; k += NT) hist[k] = 0;
    if (f.hslot >= 0) {  // the global histogram of the first pass is discarded: zero it for the next run
      uint4* gh = reinterpret_cast<uint4*>(a.hist + (uint64_t)f.hslot * 2 * ND);
      for (int k = tid; k < 2 * ND / 4; k += NT) gh[k] = make_uint4(0, 0, 0, 0);
    }
    if (tid == 0) k3.cursor = 0;
    __syncthreads();
    {
      const int lane = tid & 31, w = tid >> 5;
      if (w < UNITS) {
        uint2* stage = reinterpret_cast<uint2*>(gbuf) + w * UE;
        uint32_t mk = 0, clo = 0, dmin = 0, dmax = 0;
        for (uint32_t c = f.ch0; c < f.ch0 + f.nch; ++c) {
          uint32_t e0, n;
          unit_span(a, f, c, (uint32_t)w, e0, n);
          uint32_t cnt = 0;
          if (n) {
            Raw r;
            load_unit(f.x, f.dtype, e0, n, r);
            cnt = classify_any(f.dtype, r, e0, n, lo, lo_neg, lo != lo_neg, stage, clo);
          }
          uint32_t off = 0;
          if (lane == 0) {
            off = atomicAdd(&k3.cursor, cnt);
            a.u_off[(uint64_t)c * UNITS + w] = off;
            a.u_cnt[(uint64_t)c * UNITS + w] = cnt;
          }
          off = __shfl_sync(0xFFFFFFFFu, off, 0);
          __syncwarp();
          emit_unit(stage, cnt, le(a, f) + off, hist, mk, dmin, dmax);
          __syncwarp();
        }
      }
    }
    __syncthreads();
    ncand = k3.cursor;
    hist_ok = true;
    if (f.hslot >= 0) {  // later phases reload the histogram of the re-streamed list
      uint4* gh = reinterpret_cast<uint4*>(a.hist + (uint64_t)f.hslot * 2 * ND);
      const uint4* h4 = reinterpret_cast<const uint4*>(hist);
      for (int k = tid; k < 2 * ND / 4; k += NT) gh[k] = h4[k];
    }
  } else if (f.hslot >= 0) {
    const uint4* gh = reinterpret_cast<const uint4*>(a.hist + (uint64_t)f.hslot * 2 * ND);
    uint4* h4 = reinterpret_cast<uint4*>(hist);
    for (int k = tid; k < 2 * ND / 4; k += NT) h4[k] = __ldcg(gh + k);
    hist_ok = true;
  }
  const List L = (FUSED && Lin) ? *Lin : List{nullptr, le(a, f), 0};
  if (!hist_ok) {
    for (int k = tid; k < 2 * ND; k += NT) hist[k] = 0;
    __syncthreads();
    list_foreach<NT, LU>(L, ncand, [&](uint32_t b, uint32_t, bool v) {
      if (v) atomicAdd(&hist[((b >> 31) ? ND : 0) + ((b & 0x7FFFFFFFu) >> DSH)], 1u);
    });
  }
  __syncthreads();
  prof_mark(a, ifi, 1);
  // candidates with key != 0 (only lo == 0 admits zeros)
  uint64_t cnt_nz = ncand;
  if (PH == 1) cnt_nz = st.cnt_nz;
  else if (lo == 0) {
    cnt_nz = (uint64_t)ncand - hist[0] - hist[ND];  // digit 0 holds zeros and tiny values
    uint32_t tiny = 0;
    list_foreach<NT, LU>(L, ncand, [&](uint32_t b, uint32_t, bool v) {
      const uint32_t key = b & 0x7FFFFFFFu;
      tiny += (v && key != 0 && (key >> DSH) == 0) ? 1u : 0u;
    });
    tiny = __reduce_add_sync(0xFFFFFFFFu, tiny);
    if (tid == 0) k3.cnt_nz = 0;
    __syncthreads();
    if ((tid & 31) == 0) atomicAdd((unsigned long long*)&k3.cnt_nz, (unsigned long long)tiny);
    __syncthreads();
    cnt_nz += k3.cnt_nz;
    __syncthreads();
  }
  // (NOCLS instantiations serve encode batches only: lo >= 1 there, so no zero mode)
  const bool zero_mode = !NOCLS && kk > 0 && lo == 0;
  const bool keep_none = kk == 0;
  const bool only_nonzero = kk > 0 && cnt_nz < kk && !zero_mode;
  auto hash_of = [seed](uint32_t, uint32_t x) -> uint64_t { return splitmix(seed, x); };
  auto key31 = [](uint32_t b) -> uint64_t { return b & 0x7FFFFFFFu; };
  auto all_pred = [](uint32_t, uint32_t) { return true; };
  uint32_t tau_key = 0;
  uint64_t ck_star = 0, h_star = 0;
  bool tie_all = true;
  int dtau = -1;  // digit of tau on the fast path (-1: every candidate bin counts fully)
  // NOCLS: a lambda = 0 encode batch; the class-select, zero-mode and ATKF-only output code
  // is compiled out of this instantiation
  const bool use_cls = !NOCLS && a.lam > 0.0 && kk > 0 && !only_nonzero;
  const bool fast = !zero_mode && !use_cls;
  // lambda > 0 outside zero mode: tau, the class select and the MS cuts are all bracketed
  // by digit histograms and resolved inside gathered bins (a few passes over the list)
  const bool cls_fast = use_cls && !zero_mode && !FUSED && PH == 0;
  List A{reinterpret_cast<uint2*>(gbuf), me(a, f), GSM};
  uint32_t nA = 0;
  if (kk > 0 && !only_nonzero) {
    if (zero_mode && cnt_nz < kk) {
      // tau == 0 (ATKF-only mode): every nonzero is kept; choose kk - nnz zeros by hash
      const SelRes s = select_exact<NT, LU>(sh, scratch, L, ncand, all_pred, key31, hash_of, 0, 1, kk - cnt_nz);
      h_star = s.sec;
      tie_all = s.all_ties;
    } else if (!fast && !cls_fast) {
      const uint64_t klo = lo_neg < lo ? lo_neg : lo;
      const SelRes s = select_exact<NT, LU>(sh, scratch, L, ncand, all_pred, key31, hash_of, klo,
                                        (uint64_t)st.maxkey + 1, kk);
      tau_key = s.key;
      ck_star = s.key;
      h_star = s.sec;
      tie_all = s.all_ties;
    } else {
      prof_mark(a, ifi, 2);
      if (!FUSED && PH == 0 && fast && a.big_ncand && ncand > a.big_ncand) {
        // digit of tau over both signs; its bin is gathered by enc_gather<1> (all SMs)
        uint32_t* comb = scratch;
        for (int k = tid; k < ND; k += NT) comb[k] = hist[k] + hist[ND + k];
        __syncthreads();
        find_digit<NT>(sh, comb, ND, kk);
        const uint32_t dt = sh.fd_digit;
        const uint64_t rt0 = kk - sh.fd_above;
        __syncthreads();
        // regions of the gather area filled by enc_gather<1>: tau's bin of both signs (0, 1,
        // contiguous), then every bin that can hold an MS cut.  A plane's kept count is
        // n_lo .. n_hi (tau's bin kept partly), so cut j lies at plane rank
        // j*floor(n_lo/M)+1 .. j*floor(n_hi/M)+1; the bins above tau's that this range touches
        // are gathered now, so the cut-bin gather pass (enc_gather<2>) is usually not needed
        if (tid == 0) {
          st.reg_key[0] = dt; st.reg_off[0] = 0; st.reg_cnt[0] = 0;
          st.reg_key[1] = ND + dt; st.reg_off[1] = hist[dt]; st.reg_cnt[1] = 0;
          k3.pend_n = 2;
          k3.cursor = hist[dt] + hist[ND + dt];
        }
        const int mcfg2[2] = {a.m_plus, a.m_minus};
        const int cap = MAXREG - 2 - (a.m_plus + a.m_minus);  // room left for PH1 (checked below)
        for (int sg = 0; sg < 2; ++sg) {
          uint32_t acc = 0;
          for (int d = tid; d < ND; d += NT) acc += (uint32_t)d > dt ? hist[sg * ND + d] : 0u;
          acc = __reduce_add_sync(0xFFFFFFFFu, acc);
          if (tid == 0) k3.s.cnt[sg] = 0;
          __syncthreads();
          if ((tid & 31) == 0) atomicAdd(&k3.s.cnt[sg], acc);
          __syncthreads();
          const uint64_t n_lo = k3.s.cnt[sg], n_hi = n_lo + hist[sg * ND + dt];
          const uint64_t M = (uint64_t)mcfg2[sg];
          if (M < 2 || n_lo < M || cap < 2) continue;
          for (uint64_t j = 1; j < M; ++j) {
            const uint64_t ra = j * (n_lo / M) + 1, rb = min(j * (n_hi / M) + 1, n_lo);
            if (ra > n_lo) continue;  // in tau's bin: gathered already
            find_digit<NT>(sh, hist + sg * ND, ND, ra);
            const uint32_t da = sh.fd_digit;
            __syncthreads();
            find_digit<NT>(sh, hist + sg * ND, ND, rb);
            const uint32_t db = sh.fd_digit;
            __syncthreads();
            if (tid == 0)
              for (uint32_t d = db; d <= da; ++d) {
                if (d <= dt || hist[sg * ND + d] == 0) continue;
                const uint32_t key = (uint32_t)sg * ND + d;
                uint32_t g = 2;
                while (g < k3.pend_n && st.reg_key[g] != key) ++g;
                if (g == k3.pend_n && g < 2u + (uint32_t)cap) {
                  st.reg_key[g] = key; st.reg_off[g] = k3.cursor; st.reg_cnt[g] = 0;
                  k3.cursor += hist[key];
                  ++k3.pend_n;
                }
              }
            __syncthreads();
          }
        }
        if (tid == 0) {
          st.dtau = (int32_t)dt;
          st.rt = rt0;
          st.nA = 0;
          st.sel_lo = lo;
          st.ncand = ncand;
          st.cnt_nz = cnt_nz;
          st.nreg = k3.pend_n;
          st.nreg_pre = k3.pend_n;
          st.reg_first = 0;
          st.pre_end = k3.cursor;
          st.sel_phase = 1;
          a.big_list[atomicAdd(&a.big_list[a.n], 1u)] = (uint32_t)ifi;  // the gathers visit these IFs only
        }
        return;
      }
      uint64_t rt;
      if (PH == 1) {
        dtau = st.dtau;
        rt = st.rt;
        nA = st.reg_cnt[0] + st.reg_cnt[1];  // tau's bin of both signs (regions 0, 1; contiguous)
        // the gathered bin: first GSM entries in shared memory, the rest read from global
        const uint2* gsrc = me(a, f);
        uint2* sdst = reinterpret_cast<uint2*>(gbuf);
        const uint32_t ns = nA < (uint32_t)GSM ? nA : (uint32_t)GSM;
        for (uint32_t k = tid; k < ns; k += NT) sdst[k] = __ldcg(gsrc + k);
        A.g = me(a, f) + GSM;
        __syncthreads();
      } else {
        // small IF: digit of tau and its bin gathered by this CTA
        uint32_t* comb = scratch;
        for (int k = tid; k < ND; k += NT) comb[k] = hist[k] + hist[ND + k];
        __syncthreads();
        find_digit<NT>(sh, comb, ND, kk);
        dtau = (int)sh.fd_digit;
        rt = kk - sh.fd_above;
        if (tid == 0) k3.nA = 0;
        __syncthreads();
        list_foreach<NT, LU>(L, ncand, [&](uint32_t b, uint32_t x, bool v) {
          if (v && ((b & 0x7FFFFFFFu) >> DSH) == (uint32_t)dtau) A.set(atomicAdd(&k3.nA, 1u), b, x);
        });
        __syncthreads();
        nA = k3.nA;
      }
      const SelRes s = select_exact<NT, LU>(sh, scratch, A, nA, all_pred, key31, hash_of, (uint64_t)dtau << DSH,
                                        (uint64_t)(dtau + 1) << DSH, rt);
      tau_key = s.key;
      ck_star = s.key;
      h_star = s.sec;
      tie_all = s.all_ties;
    }
  }
  prof_mark(a, ifi, 3);
  const double tau = kk > 0 ? (double)__uint_as_float(tau_key) : (double)__uint_as_float(st.maxkey);
  const double tau_p = __dmul_rn(__dadd_rn(1.0, a.lam), tau);
  const double tau_m = -__dmul_rn(__dsub_rn(1.0, a.lam), tau);
  // strict classes (atkf.py:72-75) as key thresholds: x > tau_p <=> key(x) > kp for x > 0,
  // x < tau_m <=> key(x) > km for x < 0 (kp, km = float keys of tau_p, |tau_m| rounded down)
  const uint32_t kp = __float_as_uint(__double2float_rd(tau_p));
  const uint32_t km = __float_as_uint(__double2float_rd(-tau_m));
  auto ckey = [kp, km](uint32_t b) -> uint64_t {
    const uint32_t key = b & 0x7FFFFFFFu;
    return ((key > ((b >> 31) ? km : kp)) ? (1ull << 31) : 0ull) | (uint64_t)key;
  };
  if (use_cls && !cls_fast) {
    const SelRes s = select_exact<NT, LU>(sh, scratch, L, ncand, all_pred, ckey, hash_of, 0, 1ull << 32, kk);
    ck_star = s.key;
    h_star = s.sec;
    tie_all = s.all_ties;
  } else if (cls_fast) {
    // the kk-th element of the order (strict first, |x| desc, hash asc) (atkf.py:77-84):
    // strict count S from the per-sign histograms plus exact counts of the two boundary
    // bins (one pass); then the class holding rank kk, the digit holding it (class-restricted
    // histogram), that bin gathered (one pass) and the element selected inside it
    const uint32_t dp = kp >> DSH, dm = km >> DSH;
    if (tid < 2) k3.keptA[tid] = 0;
    __syncthreads();
    {
      uint32_t c0 = 0, c1 = 0;
      list_foreach<NT, LU>(L, ncand, [&](uint32_t b, uint32_t, bool v) {
        const uint32_t key = b & 0x7FFFFFFFu;
        if (!v) return;
        if (b >> 31) c1 += ((key >> DSH) == dm && key > km) ? 1u : 0u;
        else c0 += ((key >> DSH) == dp && key > kp) ? 1u : 0u;
      });
      c0 = __reduce_add_sync(0xFFFFFFFFu, c0);
      c1 = __reduce_add_sync(0xFFFFFFFFu, c1);
      if ((tid & 31) == 0) { atomicAdd(&k3.keptA[0], c0); atomicAdd(&k3.keptA[1], c1); }
    }
    __syncthreads();
    const uint32_t bp = k3.keptA[0], bm = k3.keptA[1];  // strict members of the boundary bins
    uint32_t* cnt = scratch;                           // class-restricted digit counts (ND)
    uint64_t S = 0;
    {
      uint32_t acc = 0;
      for (int d = tid; d < ND; d += NT)
        acc += ((uint32_t)d > dp ? hist[d] : 0u) + ((uint32_t)d > dm ? hist[ND + d] : 0u);
      acc = __reduce_add_sync(0xFFFFFFFFu, acc);
      if (tid == 0) k3.s.cnt[0] = 0;
      __syncthreads();
      if ((tid & 31) == 0) atomicAdd(&k3.s.cnt[0], acc);
      __syncthreads();
      S = (uint64_t)k3.s.cnt[0] + bp + bm;
      __syncthreads();
    }
    const bool strict_cls = S >= kk;
    const uint64_t r = strict_cls ? kk : kk - S;
    // non-strict rank kk - S lies among positives with tau <= key <= kp (every negative
    // non-strict key is <= km < tau), so its histogram counts positives only
    for (int d = tid; d < ND; d += NT) {
      uint32_t c;
      if (strict_cls)
        c = ((uint32_t)d > dp ? hist[d] : ((uint32_t)d == dp ? bp : 0u)) +
            ((uint32_t)d > dm ? hist[ND + d] : ((uint32_t)d == dm ? bm : 0u));
      else
        c = (uint32_t)d < dp ? hist[d] : ((uint32_t)d == dp ? hist[d] - bp : 0u);
      cnt[d] = c;
    }
    __syncthreads();
    find_digit<NT>(sh, cnt, ND, r);
    const uint32_t dstar = sh.fd_digit;
    const uint64_t rr = r - sh.fd_above;
    __syncthreads();
    if (tid == 0) k3.nA = 0;
    __syncthreads();
    list_foreach<NT, LU>(L, ncand, [&](uint32_t b, uint32_t x, bool v) {
      if (v && ((b & 0x7FFFFFFFu) >> DSH) == dstar) A.set(atomicAdd(&k3.nA, 1u), b, x);
    });
    __syncthreads();
    nA = k3.nA;
    const uint64_t cb = strict_cls ? (1ull << 31) : 0ull;
    const SelRes s = select_exact<NT, LU>(
        sh, scratch, A, nA, [&](uint32_t b, uint32_t) { return (ckey(b) >> 31) == (cb >> 31); }, ckey, hash_of,
        cb | ((uint64_t)dstar << DSH), cb | ((uint64_t)(dstar + 1) << DSH), rr);
    ck_star = s.key;
    h_star = s.sec;
    tie_all = s.all_ties;
  }
  auto kept_of = [&](uint32_t b, uint32_t x) -> bool {
    if (keep_none) return false;
    const uint32_t key = b & 0x7FFFFFFFu;
    if (only_nonzero) return key != 0;
    if (!zero_mode && key == 0) return false;
    const uint64_t ck = use_cls ? ckey(b) : (uint64_t)key;
    if (ck != ck_star) return ck > ck_star;
    return tie_all || splitmix(seed, x) <= h_star;
  };
  // ---- ATKF-only: kept flat indices in ascending order, tau
  if (!NOCLS && a.atkf_only) {
    int64_t* out = a.kept_out + a.kept_off[ifi];
    uint64_t run = 0;
    for (uint64_t u = (uint64_t)f.ch0 * UNITS; u < (uint64_t)(f.ch0 + f.nch) * UNITS; ++u) {
      const uint32_t off = a.u_off[u], cn = a.u_cnt[u];
      for (uint32_t base = 0; base < cn; base += NT) {
        const uint32_t j = base + tid;
        bool kp = false;
        uint32_t x = 0;
        if (j < cn) {
          const uint2 e = __ldcg(L.g + off + j);
          x = e.y;
          kp = kept_of(e.x, e.y);
        }
        uint32_t tot;
        const uint32_t ex = block_excl_scan_u32(kp ? 1u : 0u, sh.red, &tot);
        if (kp) out[run + ex] = (int64_t)x;
        run += tot;
      }
    }
    zero_hist(a, f);
    if (tid == 0) {
      st.sel_phase = 0;
      a.tau3[3 * ifi + 0] = tau;
      a.tau3[3 * ifi + 1] = tau_p;
      a.tau3[3 * ifi + 2] = tau_m;
      a.status[ifi] = SIF_OK;
    }
    return;
  }
  prof_mark(a, ifi, 4);
  // ---- kept nonzeros per sign
  uint64_t nnz[2] = {0, 0};
  if (fast) {
    if (tid < 2) k3.keptA[tid] = 0;
    __syncthreads();
    if (dtau >= 0) {
      uint32_t c0 = 0, c1 = 0;
      list_foreach<NT, LU>(A, nA, [&](uint32_t b, uint32_t x, bool v) {
        if (v && kept_of(b, x)) { if (b >> 31) ++c1; else ++c0; }
      });
      c0 = __reduce_add_sync(0xFFFFFFFFu, c0);
      c1 = __reduce_add_sync(0xFFFFFFFFu, c1);
      if ((tid & 31) == 0) { atomicAdd(&k3.keptA[0], c0); atomicAdd(&k3.keptA[1], c1); }
    }
    // per-sign histograms restricted to kept elements: bins above tau's digit count fully
    for (int k = tid; k < 2 * ND; k += NT) {
      const int d = k & (ND - 1);
      if (d < dtau) hist[k] = 0;
    }
    if (dtau >= 0 && tid < 2) hist[tid * ND + dtau] = 0;  // replaced below
    __syncthreads();
    if (dtau >= 0 && tid < 2) hist[tid * ND + dtau] = k3.keptA[tid];
    __syncthreads();
    // nnz per sign = sum of the adjusted histograms (excluding digit 0 keys == 0 never occur: lo >= 1)
    for (int s = 0; s < 2; ++s) {
      uint32_t acc = 0;
      for (int k = tid; k < ND; k += NT) acc += hist[s * ND + k];
      acc = __reduce_add_sync(0xFFFFFFFFu, acc);
      if (tid == 0) k3.s.cnt[s] = 0;
      __syncthreads();
      if ((tid & 31) == 0) atomicAdd(&k3.s.cnt[s], acc);
      __syncthreads();
      nnz[s] = k3.s.cnt[s];
      __syncthreads();
    }
    if (keep_none) { nnz[0] = 0; nnz[1] = 0; }
  } else {
    uint32_t c0 = 0, c1 = 0, m0 = 0xFFFFFFFFu, m1 = 0xFFFFFFFFu;
    list_foreach<NT, LU>(L, ncand, [&](uint32_t b, uint32_t x, bool v) {
      const uint32_t key = b & 0x7FFFFFFFu;
      if (v && key != 0 && kept_of(b, x)) {
        if (b >> 31) { ++c1; m1 = min(m1, key); } else { ++c0; m0 = min(m0, key); }
      }
    });
    c0 = __reduce_add_sync(0xFFFFFFFFu, c0);
    c1 = __reduce_add_sync(0xFFFFFFFFu, c1);
    m0 = __reduce_min_sync(0xFFFFFFFFu, m0);
    m1 = __reduce_min_sync(0xFFFFFFFFu, m1);
    if (tid < 2) { k3.s.cnt[tid] = 0; k3.s.cnt[2 + tid] = 0xFFFFFFFFu; }
    __syncthreads();
    if ((tid & 31) == 0) {
      atomicAdd(&k3.s.cnt[0], c0); atomicAdd(&k3.s.cnt[1], c1);
      atomicMin(&k3.s.cnt[2], m0); atomicMin(&k3.s.cnt[3], m1);
    }
    __syncthreads();
    nnz[0] = k3.s.cnt[0];
    nnz[1] = k3.s.cnt[1];
    if (cls_fast) {
      // per sign the kept set is a magnitude-top set: every
      // candidate above the digit of its smallest kept key is kept, that digit partially;
      // the histograms become kept histograms (the partial bins' full sizes are kept for
      // sizing the cut gathers)
      const uint32_t dl[2] = {k3.s.cnt[2] >> DSH, k3.s.cnt[3] >> DSH};
      __syncthreads();
      for (int sg = 0; sg < 2; ++sg) {
        uint32_t above = 0;
        for (int d = tid; d < ND; d += NT) above += ((uint32_t)d > dl[sg] && nnz[sg]) ? hist[sg * ND + d] : 0u;
        above = __reduce_add_sync(0xFFFFFFFFu, above);
        if (tid == 0) k3.s.cnt[4 + sg] = 0;
        __syncthreads();
        if ((tid & 31) == 0) atomicAdd(&k3.s.cnt[4 + sg], above);
        __syncthreads();
        const uint32_t part = nnz[sg] ? (uint32_t)nnz[sg] - k3.s.cnt[4 + sg] : 0u;
        if (tid == 0) k3.fullb[sg] = nnz[sg] ? hist[sg * ND + dl[sg]] : 0u;
        __syncthreads();
        for (int d = tid; d < ND; d += NT) {
          if (!nnz[sg] || (uint32_t)d < dl[sg]) hist[sg * ND + d] = 0;
          else if ((uint32_t)d == dl[sg]) hist[sg * ND + d] = part;
        }
        if (tid == 0) k3.lowd[sg] = nnz[sg] ? dl[sg] : 0xFFFFFFFFu;
        __syncthreads();
      }
    }
    __syncthreads();
  }
  prof_mark(a, ifi, 5);
  // ---- MS cuts (msplit.py:68-80): element at rank j*base of each sign plane
  const int mcfg[2] = {a.m_plus, a.m_minus};
  uint64_t meff[2], base[2];
  for (int s = 0; s < 2; ++s) {
    const uint64_t m = (uint64_t)mcfg[s];
    meff[s] = nnz[s] < m ? nnz[s] : m;
    if (meff[s] < 1) meff[s] = 1;
    base[s] = nnz[s] / meff[s];
  }
  const int B = (int)(meff[0] + meff[1]);
  const int ncut0 = (int)meff[0] - 1;
  const int ncut = B - 2;
  bool use_reg = false;   // PH 1: pending cut bins go to the all-SM gathers (enc_gather<2>)
  bool cls_hand = false;  // PH 0, lambda > 0: the same, set up here
  if (fast || cls_fast) {
    // digit of every cut from the kept histograms; cuts in tau's bin resolve from A
    if (tid == 0) k3.pend_n = 0;
    __syncthreads();
    for (int ci = 0; ci < ncut; ++ci) {
      const uint32_t s = ci < ncut0 ? 0u : 1u;
      const int j = (s == 0 ? ci : ci - ncut0) + 1;
      const uint64_t r1 = (uint64_t)j * base[s] + 1;
      find_digit<NT>(sh, hist + s * ND, ND, r1);
      const uint32_t dc = sh.fd_digit;
      const uint64_t rc = r1 - sh.fd_above;
      if (fast && (int)dc == dtau) {
        const SelRes r = select_exact<NT, LU>(
            sh, scratch, A, nA, [&](uint32_t b, uint32_t x) { return (b >> 31) == s && kept_of(b, x); }, key31,
            [](uint32_t, uint32_t x) -> uint64_t { return x; }, (uint64_t)dc << DSH, (uint64_t)(dc + 1) << DSH, rc,
            31);
        if (tid == 0) { st.cut_key[ci] = r.key; st.cut_idx[ci] = (uint32_t)r.sec; }
      } else if (tid == 0) {
        const uint32_t p = k3.pend_n++;
        k3.pend_s[p] = s; k3.pend_d[p] = dc; k3.pend_r[p] = (uint32_t)rc; k3.pend_ci[p] = (uint32_t)ci;
      }
      __syncthreads();
    }
    prof_mark(a, ifi, 6);
    const uint32_t np = k3.pend_n;
    // the all-SM gathers hold one region per lane: more distinct cut bins than MAXREG
    // (many blocks) are gathered in this CTA instead
    if (PH == 1 && np > 0) {
      if (tid == 0) {
        uint32_t nreg = st.nreg_pre;
        for (uint32_t p = 0; p < np; ++p) {
          const uint32_t d = k3.pend_s[p] * ND + k3.pend_d[p];
          bool seen = false;
          for (uint32_t g = 2; g < st.nreg_pre; ++g) seen |= st.reg_key[g] == d;
          for (uint32_t q = 0; q < p; ++q) seen |= k3.pend_s[q] * ND + k3.pend_d[q] == d;
          nreg += seen ? 0u : 1u;
        }
        k3.s.cnt[0] = nreg;
      }
      __syncthreads();
      use_reg = k3.s.cnt[0] <= (uint32_t)MAXREG;
      __syncthreads();
    }
    // lambda > 0 on a large IF: the cut bins (the partial bin at the kept threshold whole)
    // go to the all-SM gather (enc_gather<2>) and one CTA per pending cut (enc_select<2>,
    // kept test from IfSt) instead of a gather pass and sequential selects in this CTA
    if (PH == 0 && cls_fast && np > 0 && a.big_ncand && ncand > a.big_ncand) {
      if (tid == 0) {
        uint32_t nreg = 0, off = 0;
        bool fits = true;
        for (uint32_t p = 0; p < np && fits; ++p) {
          const uint32_t sg = k3.pend_s[p];
          const uint32_t d = sg * ND + k3.pend_d[p];
          uint32_t g = 0;
          while (g < nreg && st.reg_key[g] != d) ++g;
          if (g == nreg) {
            if (nreg == (uint32_t)MAXREG) { fits = false; break; }
            st.reg_key[g] = d;
            st.reg_off[g] = off;
            st.reg_cnt[g] = 0;
            off += k3.pend_d[p] == k3.lowd[sg] ? k3.fullb[sg] : hist[d];
            ++nreg;
          }
          st.pend_s[p] = sg; st.pend_d[p] = k3.pend_d[p]; st.pend_r[p] = k3.pend_r[p];
          st.pend_ci[p] = k3.pend_ci[p]; st.pend_reg[p] = g;
        }
        if (fits) {
          st.nreg = nreg;
          st.reg_first = 0;
          st.pend_n = np;
          a.big_list[atomicAdd(&a.big_list[a.n], 1u)] = (uint32_t)ifi;  // the gathers visit listed IFs only
        }
        k3.s.cnt[0] = fits ? 1u : 0u;
      }
      __syncthreads();
      cls_hand = k3.s.cnt[0] != 0;
      __syncthreads();
    }
    if (cls_hand) {
      // resolved by enc_gather<2> + enc_select<2> (sel_phase 2)
    } else if (use_reg) {
      // regions of the gather area for the pending cut bins (sizes from the histogram);
      // enc_gather<2> fills them with all SMs, enc_select<2> resolves the cuts
      // bins predicted in PH 0 are already gathered; any other is appended as a new region
      // (filled by enc_gather<2>, sel_phase 2; otherwise only enc_select<2> runs, sel_phase 5)
      if (tid == 0) {
        const uint32_t npre = st.nreg_pre;
        uint32_t nreg = npre, off = st.pre_end;
        for (uint32_t p = 0; p < np; ++p) {
          const uint32_t d = k3.pend_s[p] * ND + k3.pend_d[p];
          uint32_t g = 2;
          while (g < nreg && st.reg_key[g] != d) ++g;
          if (g == nreg) {
            st.reg_key[g] = d;
            st.reg_off[g] = off;
            st.reg_cnt[g] = 0;
            off += hist[d];
            ++nreg;
          }
          st.pend_s[p] = k3.pend_s[p]; st.pend_d[p] = k3.pend_d[p]; st.pend_r[p] = k3.pend_r[p];
          st.pend_ci[p] = k3.pend_ci[p]; st.pend_reg[p] = g;
        }
        st.nreg = nreg;
        st.reg_first = npre;
        st.pend_n = np;
      }
    } else if (np > 0) {
      // gather every pending cut bin in one pass, each (sign, digit) into its own region
      // of the gather area (sizes from the histogram); A is no longer needed
      uint32_t* pm = scratch;                                         // 2*ND bits
      uint8_t* pslot = reinterpret_cast<uint8_t*>(scratch + 2 * ND / 32);  // (sign,digit) -> region
      for (int k = tid; k < 2 * ND / 32; k += NT) pm[k] = 0;
      __syncthreads();
      if (tid == 0) {
        uint32_t nreg = 0, off = 0;
        for (uint32_t p = 0; p < np; ++p) {
          const uint32_t d = k3.pend_s[p] * ND + k3.pend_d[p];
          if (!((pm[d >> 5] >> (d & 31)) & 1u)) {
            pm[d >> 5] |= 1u << (d & 31);
            pslot[d] = (uint8_t)nreg;
            k3.reg_off[nreg] = off;
            k3.reg_cnt[nreg] = 0;
            // a partial (lambda > 0) bin is gathered whole: size it by all its candidates
            const uint32_t sg = k3.pend_s[p];
            off += (cls_fast && k3.pend_d[p] == k3.lowd[sg]) ? k3.fullb[sg] : hist[d];
            ++nreg;
          }
          k3.pend_reg[p] = pslot[d];
        }
      }
      __syncthreads();
      uint2* gat = me(a, f);
      list_foreach<NT, LU>(L, ncand, [&](uint32_t b, uint32_t x, bool v) {
        const uint32_t d = ((b >> 31) ? ND : 0) + ((b & 0x7FFFFFFFu) >> DSH);
        if (v && ((pm[d >> 5] >> (d & 31)) & 1u)) {
          const uint32_t g = pslot[d];
          __stcg(gat + k3.reg_off[g] + atomicAdd(&k3.reg_cnt[g], 1u), make_uint2(b, x));
        }
      });
      __syncthreads();
      for (uint32_t p = 0; p < np; ++p) {
        if (p == 0) prof_mark(a, ifi, 7);
        const uint32_t g = k3.pend_reg[p];
        const List Bp{nullptr, gat + k3.reg_off[g], 0};
        const uint32_t dc = k3.pend_d[p];
        // a bin above the kept threshold is kept whole; lambda > 0's partial bin is filtered
        const SelRes r = select_exact<NT, LU>(
            sh, scratch, Bp, k3.reg_cnt[g], [&](uint32_t b, uint32_t x) { return !cls_fast || kept_of(b, x); }, key31,
            [](uint32_t, uint32_t x) -> uint64_t { return x; }, (uint64_t)dc << DSH, (uint64_t)(dc + 1) << DSH,
            k3.pend_r[p], 31);
        if (tid == 0) { st.cut_key[k3.pend_ci[p]] = r.key; st.cut_idx[k3.pend_ci[p]] = (uint32_t)r.sec; }
        __syncthreads();
      }
    }
  } else {
    for (int ci = 0; ci < ncut; ++ci) {
      const uint32_t s = ci < ncut0 ? 0u : 1u;
      const int j = (s == 0 ? ci : ci - ncut0) + 1;
      const uint64_t rank0 = (uint64_t)j * base[s];
      const SelRes r = select_exact<NT, LU>(
          sh, scratch, L, ncand,
          [&](uint32_t b, uint32_t x) { return (b >> 31) == s && (b & 0x7FFFFFFFu) != 0 && kept_of(b, x); }, key31,
          [](uint32_t, uint32_t x) -> uint64_t { return x; }, 1, 1ull << 31, rank0 + 1, 31);
      if (tid == 0) { st.cut_key[ci] = r.key; st.cut_idx[ci] = (uint32_t)r.sec; }
      __syncthreads();
    }
  }
  prof_mark(a, ifi, 8);
  zero_hist(a, f);
  if (tid == 0) {
    st.sel_phase = cls_hand ? 2u : (use_reg && fast) ? (st.nreg > st.nreg_pre ? 2u : 5u) : 0u;
    uint32_t fl = 0;
    if (keep_none) fl |= F_KEEP_NONE;
    if (only_nonzero) fl |= F_ONLY_NONZERO;
    if (zero_mode) fl |= F_ZERO_MODE;
    if (use_cls) fl |= F_USE_CLS;
    if (tie_all) fl |= F_TIE_ALL;
    st.flags = fl;
    st.tau_key = tau_key;
    st.ck_star = ck_star;
    st.h_star = h_star;
    st.tau = tau; st.tau_p = tau_p; st.tau_m = tau_m;
    st.nnz[0] = nnz[0]; st.nnz[1] = nnz[1];
    st.base[0] = base[0]; st.base[1] = base[1];
    st.meff0 = (uint32_t)meff[0];
    st.B = (uint32_t)B; st.ncut0 = (uint32_t)ncut0; st.ncut = (uint32_t)ncut;
    st.ncand = ncand;
  }
}

template <int PH, bool DEEP = false, bool NOCLS = false>
__global__ void __launch_bounds__(SNT) enc_select(EArgs a) {
  extern __shared__ __align__(16) uint8_t dsm_raw[];
  __shared__ K3Sh k3;
  if (a.info[blockIdx.x].path != PATH_PIPE) return;  // selected by enc_post
  select_if<PH, SNT, false, DEEP, NOCLS>(a, (int)blockIdx.x, reinterpret_cast<uint32_t*>(dsm_raw), k3);
}


// ---------------------------------------------------------------------------------------
// K3t: one warp per single-chunk IF (T <= CH, e.g. a decode-step token) on the common path
// (lambda = 0, k > 0, bracket hit, no NaN/Inf, candidates fit TCAP).  The warp sorts its
// candidates once in shared memory by the composite (|x| key desc, sign, flat index asc)
// (bitonic, syncwarp only) and reads everything enc_select computes off the sorted order:
//   tau      key at position k-1; ties (equal keys, contiguous) keep the r smallest
//            splitmix64 hashes (atkf.py:37-41, :71-84);
//   MS cuts  inside a sign plane the sorted order is (value desc, flat index asc)
//            (msplit.py:54-80), so the cut of rank j*base is found by one counting pass.
// IfSt is written exactly as enc_select writes it; enc_select<0> skips these IFs
// (sel_phase = 4).  Other IFs are left to enc_select.
constexpr int TCAP = 1024;  // candidates per IF held by one warp
constexpr int TNT = 128;    // threads per CTA (4 IFs)

// r-th largest (1-based) 64-bit value(i) over i in [i0, i1), 8-bit radix digits, one
// shared-memory histogram per warp with match_any-aggregated increments.
template <class Val>
__device__ __forceinline__ uint64_t warp_select_range(uint32_t* hist, uint32_t i0, uint32_t i1, uint64_t r,
                                                      Val val) {
  const int lane = threadIdx.x & 31;
  uint64_t prefix = 0;
  for (int shift = 56; shift >= 0; shift -= 8) {
    const uint64_t hmask = shift >= 56 ? 0ull : (~0ull << (shift + 8));
    for (int k = lane; k < 256; k += 32) hist[k] = 0;
    __syncwarp();
    for (uint32_t b = i0; b < i1; b += 32) {
      const uint32_t i = b + lane;
      uint32_t d = 0xFFFFFFFFu;
      if (i < i1) {
        const uint64_t v = val(i);
        if ((v & hmask) == prefix) d = (uint32_t)(v >> shift) & 255u;
      }
      const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
      if (d != 0xFFFFFFFFu && lane == __ffs(peers) - 1) hist[d] += __popc(peers);
      __syncwarp();
    }
    uint32_t v[8], sum = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) { v[j] = hist[255 - 8 * lane - j]; sum += v[j]; }
    const uint32_t inc = warp_incl_scan_u32(sum), exc = inc - sum;
    const bool mine = (uint64_t)exc < r && r <= (uint64_t)inc;
    uint32_t dg = 0, rr = 0;
    if (mine) {
      uint32_t acc = exc;
      bool got = false;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (!got && (uint64_t)acc + v[j] >= r) { dg = 255u - 8u * lane - j; rr = (uint32_t)(r - acc); got = true; }
        acc += v[j];
      }
    }
    const uint32_t src = __ffs(__ballot_sync(0xFFFFFFFFu, mine)) - 1;
    dg = __shfl_sync(0xFFFFFFFFu, dg, src);
    r = __shfl_sync(0xFFFFFFFFu, rr, src);
    prefix |= (uint64_t)dg << shift;
    __syncwarp();
  }
  return prefix;
}

__global__ void __launch_bounds__(TNT) enc_select_tiny(EArgs a) {
  __shared__ uint64_t srt[TNT / 32][TCAP];
  __shared__ uint32_t hst[TNT / 32][256];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int ifi = blockIdx.x * (TNT / 32) + w;
  if (ifi >= a.n) return;
  const IfInfo& f = a.info[ifi];
  IfSt& st = a.st[ifi];
  const uint64_t kk = f.kk;
  if (f.path != PATH_PIPE) return;
  const uint32_t n = st.ncand;
  if (a.atkf_only || f.hslot >= 0 || f.T > (uint64_t)CH || a.lam != 0.0 || kk == 0 || st.err ||
      st.maxkey >= kNonFiniteKey || st.lo < 1 || st.cnt_lo < kk || n > (uint32_t)TCAP || n < kk)
    return;  // enc_select handles it
  uint64_t* c = srt[w];
  uint32_t* h = hst[w];
  const uint2* L = le(a, f);
  uint32_t P = 32;
  while (P < n) P <<= 1;
  // composite: key (31 bits) | plus-sign flag | ~flat index; padding 0 sorts last
  for (uint32_t i = lane; i < P; i += 32) {
    uint64_t v = 0;
    if (i < n) {
      const uint2 e = __ldcg(L + i);
      v = ((uint64_t)(e.x & 0x7FFFFFFFu) << 33) | ((uint64_t)((e.x >> 31) ^ 1u) << 32) | (uint64_t)(~e.y);
    }
    c[i] = v;
  }
  __syncwarp();
  for (uint32_t k = 2; k <= P; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t q = lane; q < P / 2; q += 32) {
        const uint32_t i = ((q & ~(j - 1)) << 1) | (q & (j - 1)), ix = i | j;
        const uint64_t x = c[i], y = c[ix];
        const bool desc = (i & k) == 0;
        if (desc ? (x < y) : (x > y)) { c[i] = y; c[ix] = x; }
      }
      __syncwarp();
    }
  }
  auto key_at = [&](uint32_t p) -> uint32_t { return (uint32_t)(c[p] >> 33); };
  // ---- tau and its ties [G, G+E) in the sorted order
  const uint32_t tau_key = key_at((uint32_t)kk - 1);
  uint32_t gt = 0, eq = 0;
  for (uint32_t i = lane; i < n; i += 32) {
    const uint32_t k = key_at(i);
    gt += k > tau_key;
    eq += k == tau_key;
  }
  const uint32_t G = __reduce_add_sync(0xFFFFFFFFu, gt), E = __reduce_add_sync(0xFFFFFFFFu, eq);
  const uint64_t r_eq = kk - G;
  const bool tie_all = r_eq == E;
  const uint64_t seed = f.seed;
  uint64_t h_star = 0;
  if (!tie_all)  // the r_eq-th smallest hash among the ties = the r_eq-th largest ~hash
    h_star = ~warp_select_range(h, G, G + E, r_eq,
                                [&](uint32_t i) -> uint64_t { return ~splitmix(seed, ~(uint32_t)c[i]); });
  // ---- kept counts per sign and MS cuts: rank of each kept element inside its plane
  uint32_t k0 = 0, k1 = 0;
  for (uint32_t i = lane; i < n; i += 32) {
    const bool kp = i < G || (i < G + E && (tie_all || splitmix(seed, ~(uint32_t)c[i]) <= h_star));
    if (kp) { if ((c[i] >> 32) & 1u) ++k0; else ++k1; }
  }
  uint64_t nnz[2];
  nnz[0] = __reduce_add_sync(0xFFFFFFFFu, k0);
  nnz[1] = __reduce_add_sync(0xFFFFFFFFu, k1);
  const int mcfg[2] = {a.m_plus, a.m_minus};
  uint64_t meff[2], base[2];
  for (int sg = 0; sg < 2; ++sg) {
    const uint64_t m = (uint64_t)mcfg[sg];
    meff[sg] = nnz[sg] < m ? nnz[sg] : m;
    if (meff[sg] < 1) meff[sg] = 1;
    base[sg] = nnz[sg] / meff[sg];
  }
  const int B = (int)(meff[0] + meff[1]);
  const int ncut0 = (int)meff[0] - 1;
  const int ncut = B - 2;
  if (ncut > 0) {
    uint32_t run0 = 0, run1 = 0;  // kept elements of each plane before this window
    const uint32_t le_mask = 0xFFFFFFFFu >> (31 - lane);
    for (uint32_t b0 = 0; b0 < G + E; b0 += 32) {
      const uint32_t i = b0 + lane;
      bool kp = false;
      uint32_t sg = 0;
      if (i < n) {
        kp = i < G || (i < G + E && (tie_all || splitmix(seed, ~(uint32_t)c[i]) <= h_star));
        sg = ((c[i] >> 32) & 1u) ? 0u : 1u;
      }
      const uint32_t m0 = __ballot_sync(0xFFFFFFFFu, kp && sg == 0), m1 = __ballot_sync(0xFFFFFFFFu, kp && sg == 1);
      if (kp) {
        const uint64_t rank = (uint64_t)(sg == 0 ? run0 + __popc(m0 & le_mask) : run1 + __popc(m1 & le_mask));
        const uint64_t bs = base[sg];
        // rank j*base + 1 (1-based) starts block j, j = 1 .. meff-1
        if (bs > 0 && (rank - 1) % bs == 0) {
          const uint64_t j = (rank - 1) / bs;
          if (j >= 1 && j < meff[sg]) {
            const int ci = (sg == 0 ? 0 : ncut0) + (int)j - 1;
            st.cut_key[ci] = (uint32_t)(c[i] >> 33);
            st.cut_idx[ci] = ~(uint32_t)c[i];
          }
        }
      }
      run0 += __popc(m0);
      run1 += __popc(m1);
    }
  }
  if (lane == 0) {
    const double tau = (double)__uint_as_float(tau_key);
    st.flags = tie_all ? F_TIE_ALL : 0u;
    st.tau_key = tau_key;
    st.ck_star = tau_key;
    st.h_star = h_star;
    st.tau = tau;
    st.tau_p = __dmul_rn(__dadd_rn(1.0, a.lam), tau);
    st.tau_m = -__dmul_rn(__dsub_rn(1.0, a.lam), tau);
    st.nnz[0] = nnz[0]; st.nnz[1] = nnz[1];
    st.base[0] = base[0]; st.base[1] = base[1];
    st.meff0 = (uint32_t)meff[0];
    st.B = (uint32_t)B; st.ncut0 = (uint32_t)ncut0; st.ncut = (uint32_t)ncut;
    st.ncand = n;
    st.sel_phase = 4;  // resolved here; enc_select<0> skips the IF
  }
}

// ---------------------------------------------------------------------------------------
// Per-IF kept test and block id, evaluated by the chunk kernels from IfSt.
struct KeptCtx {
  uint32_t flags;
  uint64_t ck_star, h_star, seed;
  double tau_p, tau_m;
  int ncut0, ncut, meff0;
  uint32_t ck[MAXB], cx[MAXB];
  __device__ __forceinline__ bool kept(uint32_t b, uint32_t x) const {
    const uint32_t key = b & 0x7FFFFFFFu;
    if (key == 0) return false;  // planes hold nonzeros only (msplit.py:48-51)
    if (flags & F_KEEP_NONE) return false;
    if (flags & F_ONLY_NONZERO) return true;
    uint64_t c = key;
    if (flags & F_USE_CLS) {
      const double v = (double)__uint_as_float(b);
      if (v > tau_p || v < tau_m) c |= 1ull << 31;
    }
    if (c != ck_star) return c > ck_star;
    return (flags & F_TIE_ALL) || splitmix(seed, x) <= h_star;
  }
  __device__ __forceinline__ int block_of(uint32_t b, uint32_t x) const {
    const uint32_t key = b & 0x7FFFFFFFu;
    const int s = (int)(b >> 31);
    const int c0 = s ? ncut0 : 0, cn = s ? ncut : ncut0;
    int blk = 0;
    for (int cc = c0; cc < cn; ++cc) {
      const uint32_t k2 = ck[cc];
      if (key < k2 || (key == k2 && x >= cx[cc])) ++blk;
      else break;
    }
    return (s ? meff0 : 0) + blk;
  }
};

__device__ __forceinline__ void load_kept_ctx(KeptCtx& k, const IfSt& st, uint64_t seed) {
  k.flags = st.flags;
  k.ck_star = st.ck_star;
  k.h_star = st.h_star;
  k.seed = seed;
  k.tau_p = st.tau_p;
  k.tau_m = st.tau_m;
  k.ncut0 = (int)st.ncut0;
  k.ncut = (int)st.ncut;
  k.meff0 = (int)st.meff0;
  for (int c = 0; c < k.ncut; ++c) { k.ck[c] = st.cut_key[c]; k.cx[c] = st.cut_idx[c]; }
}

// ---------------------------------------------------------------------------------------
// Chunk-kernel work split: global warp gw of GW owns chunks [nch*gw/GW, nch*(gw+1)/GW).
__device__ __forceinline__ void warp_range(const EArgs& a, uint32_t& c0, uint32_t& c1) {
  const uint64_t GW = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t gw = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  c0 = (uint32_t)((uint64_t)a.nch * gw / GW);
  c1 = (uint32_t)((uint64_t)a.nch * (gw + 1) / GW);
}

// ---------------------------------------------------------------------------------------
// Chunk-parallel gathers for enc_select (one warp per chunk, all SMs): G = 1 copies the
// candidates in tau's digit (either sign) to the IF's gather area, G = 2 copies the
// candidates of every pending (sign, digit) cut bin to its region.  Appends are
// warp-aggregated (one atomic per region per window).
template <int G>
__global__ void __launch_bounds__(CNT) enc_gather(EArgs a) {
  constexpr uint32_t LCAP = 2048;  // listed IFs whose chunk prefix fits shared memory
  __shared__ uint32_t lpre[LCAP + 1];
  __shared__ uint32_t scan_s[33];
  const int lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  const uint32_t GW = gridDim.x * (CNT / 32), gw = blockIdx.x * (CNT / 32) + (threadIdx.x >> 5);
  const uint32_t nbig = min(a.big_list[a.n], LCAP);
  // only the IFs on the multi-kernel path (big_list): their chunks, concatenated, are split
  // into one contiguous range per warp (balanced whatever the mix of IF sizes)
  if (threadIdx.x == 0) lpre[0] = 0;
  __syncthreads();  // lpre[0] is read below even when no IF is listed (nbig == 0)
  for (uint32_t b0 = 0; b0 < nbig; b0 += CNT) {
    const uint32_t li = b0 + threadIdx.x;
    const uint32_t v = li < nbig ? a.info[a.big_list[li]].nch : 0u;
    uint32_t tot;
    const uint32_t ex = block_excl_scan_u32(v, scan_s, &tot);
    if (li < nbig) lpre[li + 1] = lpre[b0] + ex + v;
    __syncthreads();
  }
  // every IF listed (e.g. a batch of prefill IFs): plain contiguous ranges over all chunks;
  // otherwise contiguous ranges over the concatenated chunks of the listed IFs
  const bool all = a.big_list[a.n] >= (uint32_t)a.n;
  const uint32_t V = all ? (uint32_t)a.nch : lpre[nbig];
  const uint32_t v0 = (uint32_t)((uint64_t)V * gw / GW), v1 = (uint32_t)((uint64_t)V * (gw + 1) / GW);
  uint32_t li = 0;
  if (!all) {
    uint32_t lo = 0, hi = nbig;  // last li with lpre[li] <= v0
    while (lo + 1 < hi) { const uint32_t mid = (lo + hi) >> 1; if (lpre[mid] <= v0) lo = mid; else hi = mid; }
    li = lo;
  }
  uint32_t nreg = 0, rkey = 0xFFFFFFFFu, roff = 0;
  for (uint32_t v = v0; v < v1 && (all || li < nbig); ++li) {
   uint32_t ifi, vb, vend, cbeg, cend;
   if (all) {
     ifi = a.ch_if[v];
     vb = v;
     vend = min(v1, a.info[ifi].ch0 + a.info[ifi].nch);
     cbeg = vb;
     cend = vend;
   } else {
     ifi = a.big_list[li];
     vb = v;
     vend = min(v1, lpre[li + 1]);
     cbeg = a.info[ifi].ch0 + (vb - lpre[li]);
     cend = a.info[ifi].ch0 + (vend - lpre[li]);
   }
   v = vend;
   IfSt& st = a.st[ifi];
   if (st.sel_phase != (uint32_t)G) continue;
   const IfInfo& f = a.info[ifi];
   {
     // regions to fill: <1> every region set up by enc_select<0>, <2> the ones enc_select<1> added
     const uint32_t first = G == 1 ? 0u : st.reg_first;
     nreg = st.nreg;
     rkey = (lane < (int)nreg && (G == 1 || (uint32_t)lane >= first)) ? st.reg_key[lane] : 0xFFFFFFFFu;
     roff = lane < (int)nreg ? st.reg_off[lane] : 0u;
   }
   const uint2* gl = le(a, f);
   uint2* gat = me(a, f);
   for (uint32_t c = cbeg; c < cend; ++c) {
    const uint32_t my_uo = lane < UNITS ? a.u_off[(uint64_t)c * UNITS + lane] : 0u;
    const uint32_t my_un = lane < UNITS ? a.u_cnt[(uint64_t)c * UNITS + lane] : 0u;
    for (int u = 0; u < UNITS; ++u) {
      const uint32_t uo = __shfl_sync(0xFFFFFFFFu, my_uo, u), un = __shfl_sync(0xFFFFFFFFu, my_un, u);
      for (uint32_t j0 = 0; j0 < un; j0 += 64) {
        uint2 ev[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t j = j0 + 32 * h + lane;
          ev[h] = j < un ? __ldg(gl + uo + j) : make_uint2(0, 0);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t j = j0 + 32 * h + lane;
          const uint2 e = ev[h];
          const uint32_t dig = (e.x & 0x7FFFFFFFu) >> DSH;
          int g = -1;
          {
            const uint32_t key = j < un ? ((e.x >> 31) ? (uint32_t)ND : 0u) + dig : 0xFFFFFFFEu;
            for (uint32_t k = 0; k < nreg; ++k)
              if (__shfl_sync(0xFFFFFFFFu, rkey, (int)k) == key) g = (int)k;
          }
          {
            const uint32_t peers = __match_any_sync(0xFFFFFFFFu, g);
            const uint32_t ld = (uint32_t)(__ffs(peers) - 1);
            uint32_t base = 0;
            if (g >= 0 && lane == ld) base = atomicAdd(&st.reg_cnt[g], (uint32_t)__popc(peers));
            base = __shfl_sync(0xFFFFFFFFu, base, (int)ld);
            const uint32_t off = __shfl_sync(0xFFFFFFFFu, roff, g >= 0 ? g : 0);
            if (g >= 0) __stcg(gat + off + base + __popc(peers & lt), e);
          }
        }
      }
    }
  }
  }
}


// ---------------------------------------------------------------------------------------
// K4: one warp per chunk: kept test, block id, per-block count / min / max / last row, and
// a stable regroup of the chunk's members by block into the member slot (CSR order inside a
// block = flat order).  Also zeroes this chunk's share of the IF's output buffer.
struct K4W {
  uint32_t cnt[MAXB], mn[MAXB], mx[MAXB], xl[MAXB], pos[MAXB];
};

__global__ void __launch_bounds__(CNT, 6) enc_members(EArgs a) {
  __shared__ KeptCtx kcs[CNT / 32];
  __shared__ K4W wst[CNT / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  KeptCtx& kc = kcs[w];
  K4W& ws = wst[w];
  uint32_t c0, c1;
  warp_range(a, c0, c1);
  uint32_t cur = 0xFFFFFFFFu;
  int B = 0;
  FastDiv fk;
  fk.init(1);
  for (uint32_t c = c0; c < c1; ++c) {
    const uint32_t ifi = a.ch_if[c];
    const IfInfo& f = a.info[ifi];
    IfSt& st = a.st[ifi];
    if (st.err || f.path != PATH_PIPE) continue;
    if (ifi != cur) {
      __syncwarp();
      if (lane == 0) {
        kc.flags = st.flags; kc.ck_star = st.ck_star; kc.h_star = st.h_star; kc.seed = f.seed;
        kc.tau_p = st.tau_p; kc.tau_m = st.tau_m;
        kc.ncut0 = (int)st.ncut0; kc.ncut = (int)st.ncut; kc.meff0 = (int)st.meff0;
      }
      const int nc = (int)st.ncut;
      for (int k = lane; k < nc; k += 32) { kc.ck[k] = st.cut_key[k]; kc.cx[k] = st.cut_idx[k]; }
      __syncwarp();
      cur = ifi;
      B = (int)st.B;
      fk.init(f.K);
    }
    // zero this chunk's share of the output (K6/K7 write into a zeroed payload)
    {
      // chunk k of the IF zeroes the 512-byte stripes k, k + nch, k + 2*nch, ... of the output
      const uint32_t k = c - f.ch0;
      const uint32_t n16 = (uint32_t)(f.cap / 16);
      uint4* o4 = reinterpret_cast<uint4*>(f.out);
      for (uint32_t z = k * 32u + lane; z < n16; z += 32u * f.nch) o4[z] = make_uint4(0, 0, 0, 0);
      if (k + 1 == f.nch)
        for (uint64_t z = (uint64_t)n16 * 16 + lane; z < f.cap; z += 32) f.out[z] = 0;
    }
    for (int b = lane; b < B; b += 32) { ws.cnt[b] = 0; ws.mn[b] = 0x7FFFFFFFu; ws.mx[b] = 0; ws.xl[b] = 0; }
    __syncwarp();
    const uint2* gl = le(a, f);
    uint2* om = me(a, f) + (uint64_t)(c - f.ch0) * CH;
    const uint32_t my_uo = lane < UNITS ? a.u_off[(uint64_t)c * UNITS + lane] : 0u;
    const uint32_t my_un = lane < UNITS ? a.u_cnt[(uint64_t)c * UNITS + lane] : 0u;
    const uint32_t n = __reduce_add_sync(0xFFFFFFFFu, my_un);
    // one pass when every block fits a run of capacity n (B*n <= slot): block b's run starts
    // at b*n; otherwise block ids are kept and a second pass scatters into prefix runs
    const uint64_t slot = min((uint64_t)CH, f.T - (uint64_t)(c - f.ch0) * CH);  // member slot capacity
    const bool one = (uint64_t)B * n <= slot;
    uint32_t i = 0;
    // the first 64 candidates of the next unit are loaded while the current unit is processed
    uint2 nx[2];
    {
      const uint32_t uo = __shfl_sync(0xFFFFFFFFu, my_uo, 0), un = __shfl_sync(0xFFFFFFFFu, my_un, 0);
#pragma unroll
      for (int h = 0; h < 2; ++h) nx[h] = 32 * h + lane < un ? __ldcs(gl + uo + 32 * h + lane) : make_uint2(0, 0);
    }
    for (int u = 0; u < UNITS; ++u) {
      const uint32_t uo = __shfl_sync(0xFFFFFFFFu, my_uo, u), un = __shfl_sync(0xFFFFFFFFu, my_un, u);
      uint2 cu[2] = {nx[0], nx[1]};
      if (u + 1 < UNITS) {
        const uint32_t uo1 = __shfl_sync(0xFFFFFFFFu, my_uo, u + 1), un1 = __shfl_sync(0xFFFFFFFFu, my_un, u + 1);
#pragma unroll
        for (int h = 0; h < 2; ++h) nx[h] = 32 * h + lane < un1 ? __ldcs(gl + uo1 + 32 * h + lane) : make_uint2(0, 0);
      }
      for (uint32_t j0 = 0; j0 < un; j0 += 64) {
        // two windows in flight: both loads issued before either is used
        uint2 ev[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t j = j0 + 32 * h + lane;
          ev[h] = j0 == 0 ? cu[h] : (j < un ? __ldcs(gl + uo + j) : make_uint2(0, 0));
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t j = j0 + 32 * h + lane;
          const uint2 e = ev[h];
          int blk = -1;
          if (j < un) {
            if (kc.kept(e.x, e.y)) blk = kc.block_of(e.x, e.y);
          }
          const uint32_t peers = __match_any_sync(0xFFFFFFFFu, blk);
          const bool last = blk >= 0 && lane == 31 - __clz(peers);
          if (blk >= 0) {
            const uint32_t key = e.x & 0x7FFFFFFFu;
            atomicMin(&ws.mn[blk], key);
            atomicMax(&ws.mx[blk], key);
            if (one) __stcg(om + (uint32_t)blk * n + ws.cnt[blk] + __popc(peers & lt), e);
          }
          __syncwarp();
          if (last) { ws.cnt[blk] += __popc(peers); ws.xl[blk] = max(ws.xl[blk], e.y + 1u); }
          __syncwarp();
        }
      }
      i += un;
    }
    uint32_t carry = 0;
    for (int b0 = 0; b0 < B; b0 += 32) {  // blocks b0 + lane (two rounds above 32 blocks)
      const int b = b0 + lane;
      const uint32_t cnt = b < B ? ws.cnt[b] : 0u;
      const uint32_t sinc = warp_incl_scan_u32(cnt) + carry;
      carry = __shfl_sync(0xFFFFFFFFu, sinc, 31);
      if (b < B) {
        const uint32_t rs = one ? (uint32_t)b * n : sinc - cnt;
        ws.pos[b] = rs;
        const uint64_t ci = (uint64_t)c * a.maxb + b;
        a.ch_bcnt[ci] = cnt;
        a.ch_brs[ci] = rs;
        a.ch_blast[ci] = ws.xl[b] ? (int32_t)fk.div(ws.xl[b] - 1u) : -1;
        if (cnt) {
          atomicMin(&st.bmin[b], ws.mn[b]);
          atomicMax(&st.bmax[b], ws.mx[b]);
          atomicAdd(&st.bcount[b], cnt);
        }
      }
    }
    __syncwarp();
    if (one) continue;
    // pass 2: stable scatter into block runs of the member slot
    i = 0;
    for (int u = 0; u < UNITS; ++u) {
      const uint32_t uo = __shfl_sync(0xFFFFFFFFu, my_uo, u), un = __shfl_sync(0xFFFFFFFFu, my_un, u);
      for (uint32_t j0 = 0; j0 < un; j0 += 64) {
        uint2 ev[2];
        int bv[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // block ids recomputed (the two-pass case is rare)
          const uint32_t j = j0 + 32 * h + lane;
          ev[h] = j < un ? __ldg(gl + uo + j) : make_uint2(0, 0);
          bv[h] = (j < un && kc.kept(ev[h].x, ev[h].y)) ? kc.block_of(ev[h].x, ev[h].y) : -1;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int blk = bv[h];
          const uint32_t peers = __match_any_sync(0xFFFFFFFFu, blk);
          if (blk >= 0) {
            const uint32_t dst = ws.pos[blk] + __popc(peers & lt);
            __stcg(om + dst, ev[h]);
          }
          __syncwarp();
          if (blk >= 0 && lane == 31 - __clz(peers)) ws.pos[blk] += __popc(peers);
          __syncwarp();
        }
      }
      i += un;
    }
  }
}

// ---------------------------------------------------------------------------------------
// K5: ABQ distortion sums S[b][q] = sum |code_qbit >> (qbit - q) - code_q| (quant.py:88-99),
// one warp per chunk, over block runs.  Pass A (first_pass=1) computes q = q_bit-1 only,
// which decides most blocks (the descent stops at the first violation, quant.py:110-115);
// pass B computes every q < q_bit-1 for the blocks whose q_bit-1 distortion is within
// delta.  Per-warp accumulators in SMEM are flushed when the warp moves to another IF.
struct AbqPar {
  double vmin;
  double o[17];
  double inv[17];
  uint32_t act;
};

template <int FIRST, bool WIDE>  // WIDE: more than 32 blocks per IF in the batch
__global__ void __launch_bounds__(CNT, 4) enc_abq(EArgs a) {
  extern __shared__ __align__(16) uint8_t dsm_raw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int maxb = a.maxb, qb = a.q_bit;
  if (qb < (FIRST ? 2 : 3)) return;
  AbqPar* par = reinterpret_cast<AbqPar*>(dsm_raw) + (size_t)w * maxb;
  uint64_t* acc_s = reinterpret_cast<uint64_t*>(reinterpret_cast<AbqPar*>(dsm_raw) + (size_t)(CNT / 32) * maxb) +
                    (size_t)w * maxb * 16;
  uint32_t c0, c1;
  warp_range(a, c0, c1);
  uint32_t cur = 0xFFFFFFFFu;
  int B = 0;
  bool skipif = false;  // pass B: no block of the current IF needs the lower levels
  auto flush = [&]() {
    __syncwarp();
    if (cur != 0xFFFFFFFFu && !skipif) {
      IfSt& st = a.st[cur];
      for (int k = lane; k < B * 16; k += 32)
        if (acc_s[k]) atomicAdd((unsigned long long*)&st.S[k], (unsigned long long)acc_s[k]);
    }
    __syncwarp();
  };
  for (uint32_t c = c0; c < c1; ++c) {
    const uint32_t ifi = a.ch_if[c];
    const IfInfo& f = a.info[ifi];
    IfSt& st = a.st[ifi];
    if (st.err || f.path != PATH_PIPE) continue;
    if (ifi != cur) {
      flush();
      B = (int)st.B;
      cur = ifi;
      skipif = false;
      if (!FIRST) {  // pass B: nothing to do unless some block stays within delta at q_bit-1
        bool act = false;
        for (int b = lane; b < B; b += 32)
          if (st.bmin[b] < st.bmax[b])
            act |= !(__ddiv_rn((double)st.S[b * 16 + qb - 1], (double)st.bcount[b]) > a.delta);
        skipif = !__any_sync(0xFFFFFFFFu, act);
        if (skipif) continue;
      }
      for (int k = lane; k < B * 16; k += 32) acc_s[k] = 0;
      for (int k = lane; k < B * 16; k += 32) {
        const int b = k >> 4, q = (k & 15) + 1;
        const uint32_t m0 = st.bmin[b], m1 = st.bmax[b];
        const double vmin = (double)__uint_as_float(m0), vmax = (double)__uint_as_float(m1);
        if (q <= qb && (!FIRST || q >= qb - 1)) {  // pass A needs the scales of q_bit and q_bit-1 only
          const double o = __ddiv_rn(__dsub_rn(vmax, vmin), (double)((1u << q) - 1u));
          par[b].o[q] = o;
          par[b].inv[q] = __drcp_rn(o);
        }
        if (q == 1) {
          bool act = m0 < m1;
          if (!FIRST && act) {
            // descend past q_bit - 1 only if that level is within delta
            const double ds = __ddiv_rn((double)st.S[b * 16 + qb - 1], (double)st.bcount[b]);
            act = !(ds > a.delta);
          }
          par[b].vmin = vmin;
          par[b].act = act ? 1u : 0u;
        }
      }
      __syncwarp();
    }
    if (skipif) continue;
    // blocks in groups of 32: counts and run starts of group b0 in lane registers
    const uint64_t cb0 = (uint64_t)c * maxb;
    const uint2* gm = me(a, f) + (uint64_t)(c - f.ch0) * CH;
    const uint32_t lref = (1u << qb) - 1u;
    for (int b0 = 0; b0 < (WIDE ? B : 1); b0 += 32) {
    const uint32_t bcnt = b0 + lane < B ? a.ch_bcnt[cb0 + b0 + lane] : 0u;
    const uint32_t brs = b0 + lane < B ? a.ch_brs[cb0 + b0 + lane] : 0u;
    for (int b = b0; b < (WIDE ? min(B, b0 + 32) : B); ++b) {
      const uint32_t nb = __shfl_sync(0xFFFFFFFFu, bcnt, b - b0);
      if (nb == 0 || !par[b].act) continue;
      const uint32_t rs = __shfl_sync(0xFFFFFFFFu, brs, b - b0);
      const double vmin = par[b].vmin;
      const double oref = par[b].o[qb], iref = par[b].inv[qb];
      if (FIRST) {
        const int q = qb - 1;
        const double oq = par[b].o[q], iq = par[b].inv[q];
        uint32_t acc = 0;
        for (uint32_t i0 = 0; i0 < nb; i0 += 128) {
          uint32_t kv[4];
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const uint32_t i = i0 + 32 * h + lane;
            kv[h] = i < nb ? __ldg(&gm[rs + i].x) & 0x7FFFFFFFu : 0xFFFFFFFFu;
          }
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            if (kv[h] != 0xFFFFFFFFu) {
              const uint32_t r = quant_code(kv[h], vmin, oref, iref, lref) >> 1;
              const uint32_t cq = quant_code(kv[h], vmin, oq, iq, (1u << q) - 1u);
              acc += r > cq ? r - cq : cq - r;
            }
          }
        }
        const uint32_t v = __reduce_add_sync(0xFFFFFFFFu, acc);
        if (lane == 0) acc_s[b * 16 + q] += v;
      } else {
        uint32_t acc[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) acc[q] = 0;
        for (uint32_t i = lane; i < nb; i += 32) {
          const uint32_t key = __ldg(&gm[rs + i].x) & 0x7FFFFFFFu;
          const uint32_t cr = quant_code(key, vmin, oref, iref, lref);
#pragma unroll
          for (int q = 1; q < 15; ++q) {
            if (q < qb - 1) {
              const uint32_t cq = quant_code(key, vmin, par[b].o[q], par[b].inv[q], (1u << q) - 1u);
              const uint32_t r = cr >> (qb - q);
              acc[q] += r > cq ? r - cq : cq - r;
            }
          }
        }
#pragma unroll
        for (int q = 1; q < 15; ++q) {
          if (q < qb - 1) {
            const uint32_t v = __reduce_add_sync(0xFFFFFFFFu, acc[q]);
            if (lane == q) acc_s[b * 16 + q] += v;
          }
        }
      }
    }
    }
  }
  flush();
}

// ---------------------------------------------------------------------------------------
// K6: per-IF q*, layout, header/meta, chunk prefixes (one warp per block), row_ptr tails.
__device__ __forceinline__ void st_u32_le(uint8_t* base, uint64_t off, uint32_t v) { st_u32_le_bytes(base, off, v); }

__global__ void __launch_bounds__(256) enc_layout(EArgs a) {
  constexpr int NT = 256;
  __shared__ uint64_t s_bn[MAXB];
  __shared__ int32_t s_last[MAXB];
  __shared__ uint32_t s_q[MAXB];
  __shared__ uint64_t s_P;
  const int ifi = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const IfInfo f = a.info[ifi];
  IfSt& st = a.st[ifi];
  if (f.path != PATH_PIPE || st.err) return;
  const int B = (int)st.B;
  const uint32_t ch0 = f.ch0, nch = f.nch;
  // chunk prefixes of block b (warp b % 8): member offsets and the last row before the chunk
  for (int b = w; b < B; b += NT / 32) {
    uint32_t run = 0;
    int32_t lastp = -1;
    for (uint32_t t0 = 0; t0 < nch; t0 += 32) {
      const uint32_t k = t0 + lane;
      const uint64_t ci = (uint64_t)(ch0 + k) * a.maxb + b;
      const uint32_t v = k < nch ? a.ch_bcnt[ci] : 0u;
      const int32_t l = k < nch ? a.ch_blast[ci] : -1;
      const uint32_t inc = warp_incl_scan_u32(v);
      int32_t m = l;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xFFFFFFFFu, m, o);
        if (lane >= o) m = max(m, y);
      }
      const int32_t mex = __shfl_up_sync(0xFFFFFFFFu, m, 1);
      if (k < nch) {
        a.ch_bpre[ci] = run + inc - v;
        a.ch_bprev[ci] = max(lastp, lane ? mex : -1);
      }
      run += __shfl_sync(0xFFFFFFFFu, inc, 31);
      lastp = max(lastp, __shfl_sync(0xFFFFFFFFu, m, 31));
    }
    if (lane == 0) { s_bn[b] = run; s_last[b] = lastp; }
  }
  __syncthreads();
  // q* per block (quant.py:102-115; codec.py:176-181, :194-200)
  if (tid < B) {
    const int b = tid;
    const int s = b < (int)st.meff0 ? 0 : 1;
    const int j = s ? b - (int)st.meff0 : b;
    const uint64_t n = s_bn[b];
    const bool empty = n == 0;
    const bool degen = !empty && st.bmin[b] == st.bmax[b];
    uint32_t q;
    if (a.mode == SIF_MODE_FIXED) q = a.fixed_q[(s ? a.m_plus : 0) + j];
    else if (empty) q = (uint32_t)a.q_bit;
    else if (degen) q = 1;
    else {
      q = (uint32_t)a.q_bit;
      for (int qq = a.q_bit - 1; qq >= 1; --qq) {
        const double ds = __ddiv_rn((double)st.S[b * 16 + qq], (double)n);
        if (ds > a.delta) break;  // first violation stops the descent
        q = (uint32_t)qq;
      }
    }
    s_q[b] = q;
    st.q[b] = q;
    st.bn[b] = n;
    const double vmin = (double)__uint_as_float(st.bmin[b]), vmax = (double)__uint_as_float(st.bmax[b]);
    const double o64 = (empty || degen) ? 1.0 : __ddiv_rn(__dsub_rn(vmax, vmin), (double)((1u << q) - 1u));
    st.o64[b] = o64;
    st.inv64[b] = __drcp_rn(o64);
  }
  __syncthreads();
  if (tid == 0) {
    uint64_t pos = kHeaderBytes + (a.mode == SIF_MODE_FIXED ? (uint64_t)B : 0ull);
    for (int b = 0; b < B; ++b) {
      st.off_meta[b] = pos;
      pos += kBlockMetaBytes + 4ull * ((uint64_t)f.N + 1ull);
      st.bit_cols[b] = 8ull * pos;
      pos += (s_bn[b] * f.cb + 7ull) / 8ull;
      st.bit_codes[b] = 8ull * pos;
      pos += (s_bn[b] * s_q[b] + 7ull) / 8ull;
    }
    const uint64_t P = pos + kCrcBytes;
    st.P = P;
    s_P = P;
    if (P > f.cap) st.err = E_CAPACITY;
  }
  __syncthreads();
  const uint64_t P = s_P;
  if (P > f.cap) return;
  uint8_t* out = f.out;
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
    h[22] = (uint8_t)a.q_bit;
    h[27] = (uint8_t)a.mode;
    const uint32_t m0 = st.meff0, m1 = (uint32_t)B - st.meff0;
    h[28] = (uint8_t)m0; h[29] = (uint8_t)(m0 >> 8);
    h[30] = (uint8_t)m1; h[31] = (uint8_t)(m1 >> 8);
    for (int k = 0; k < 32; ++k) out[k] = h[k];
  }
  if (a.mode == SIF_MODE_FIXED)
    for (int b = tid; b < B; b += NT) out[kHeaderBytes + b] = (uint8_t)s_q[b];
  for (int b = tid; b < B; b += NT) {
    const uint64_t o = st.off_meta[b];
    out[o] = (uint8_t)s_q[b];
    st_u32_le(out, o + 1, __float_as_uint(s_bn[b] == 0 ? 1.0f : __double2float_rn(st.o64[b])));
    st_u32_le(out, o + 5, s_bn[b] == 0 ? 0u : st.bmin[b]);
    st_u32_le(out, o + 9, (uint32_t)s_bn[b]);
  }
  // row_ptr tails: rows after the block's last member hold nnz (msplit.py:97-100)
  for (int b = 0; b < B; ++b) {
    const uint32_t nb = (uint32_t)s_bn[b];
    if (nb == 0) continue;
    const uint64_t rp = st.off_meta[b] + kBlockMetaBytes;
    for (uint32_t r = (uint32_t)(s_last[b] + 1) + tid; r <= f.N; r += NT) st_u32_le(out, rp + 4ull * r, nb);
  }
}

// ---------------------------------------------------------------------------------------
// K7: one warp per chunk: codes at q* (quant.py:59-62), row_ptr transitions and MSB-first
// packing of cols and codes (bitstream.py:6-30).  32 consecutive fields of a block run are
// assembled into 32-bit words with shuffles; a word cut by the window end is carried into
// the next window, words at run edges are merged with atomicOr, all others stored.
struct PackPar {
  double vmin, o64, inv;
  uint64_t rp, bc, bq;
  uint32_t q, degen;
};

struct Carry {
  uint32_t W;
  uint32_t v;
};

// Pack the window of fields j0 .. j0+nv-1 (lane l holds field j0+l) of a run spanning
// payload bits [Rs, Re), width w, MSB-first (bitstream.py:12-20).  Fields are OR-ed into a
// per-warp shared-memory word buffer; words wholly inside the run are stored, words at run
// edges merged with atomicOr, and the word cut by the window end carried (cy) into the next.
__device__ __forceinline__ void pack_window(uint32_t* out32, uint32_t* buf, uint32_t val, bool valid, uint32_t w,
                                            uint32_t Rs, uint32_t Re, uint32_t j0, uint32_t nv, Carry& cy) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t P = Rs + j0 * w, E = P + nv * w;
  const bool last = E == Re;
  const uint32_t W0 = P >> 5, W1 = (E - 1) >> 5;
  const uint32_t nw = W1 - W0 + 1;
  if (lane < nw) buf[lane] = (lane == 0 && cy.W == W0) ? cy.v : 0u;
  __syncwarp();
  if (valid) {
    const uint32_t pb = P + lane * w - (W0 << 5);
    const uint32_t wi = pb >> 5, sh = pb & 31u;
    const uint64_t x = (uint64_t)val << (64u - w - sh);
    atomicOr(&buf[wi], (uint32_t)(x >> 32));
    if (sh + w > 32u) atomicOr(&buf[wi + 1], (uint32_t)x);
  }
  __syncwarp();
  const bool cut_last = ((W1 << 5) + 32 > E) && !last;  // last word continues in the next window
  const uint32_t cv = buf[nw - 1];
  if (lane < nw && !(cut_last && lane == nw - 1)) {
    const uint32_t W = W0 + lane;
    const uint32_t wv = buf[lane];
    const bool edge = (W << 5) < Rs || (W << 5) + 32 > Re;
    if (edge) { if (wv) atomicOr(out32 + W, bswap32(wv)); }
    else out32[W] = bswap32(wv);
  }
  cy.W = cut_last ? W1 : 0xFFFFFFFFu;
  cy.v = cut_last ? cv : 0u;
  __syncwarp();
}

template <bool WIDE>  // WIDE: more than 32 blocks per IF in the batch
__global__ void __launch_bounds__(CNT, 4) enc_pack(EArgs a) {
  extern __shared__ __align__(16) uint8_t dsm_raw[];
  __shared__ uint32_t pbuf[CNT / 32][2][40];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int maxb = a.maxb;
  PackPar* par = reinterpret_cast<PackPar*>(dsm_raw) + (size_t)w * maxb;
  uint32_t c0, c1;
  warp_range(a, c0, c1);
  uint32_t cur = 0xFFFFFFFFu;
  int B = 0;
  FastDiv fk;
  fk.init(1);
  for (uint32_t c = c0; c < c1; ++c) {
    const uint32_t ifi = a.ch_if[c];
    const IfInfo& f = a.info[ifi];
    IfSt& st = a.st[ifi];
    if (st.err || f.path != PATH_PIPE) continue;
    if (ifi != cur) {
      __syncwarp();
      B = (int)st.B;
      for (int b = lane; b < B; b += 32) {
        PackPar& p = par[b];
        p.vmin = (double)__uint_as_float(st.bmin[b]);
        p.o64 = st.o64[b];
        p.inv = st.inv64[b];
        p.rp = st.off_meta[b] + kBlockMetaBytes;
        p.bc = st.bit_cols[b];
        p.bq = st.bit_codes[b];
        p.q = st.q[b];
        p.degen = st.bmin[b] == st.bmax[b] ? 1u : 0u;
      }
      __syncwarp();
      cur = ifi;
      fk.init(f.K);
    }
    // blocks in groups of 32: the chunk fields of group b0 in lane registers
    for (int b0 = 0; b0 < (WIDE ? B : 1); b0 += 32) {
    const uint64_t ci = (uint64_t)c * maxb + b0 + lane;
    const bool inb = b0 + lane < B;
    const uint32_t bcnt = inb ? a.ch_bcnt[ci] : 0u;
    const uint32_t bpre = inb ? a.ch_bpre[ci] : 0u;
    const int32_t bprev = inb ? a.ch_bprev[ci] : -1;
    const uint32_t brs = inb ? a.ch_brs[ci] : 0u;
    const uint2* gm = me(a, f) + (uint64_t)(c - f.ch0) * CH;
    uint8_t* out = f.out;
    uint32_t* out32 = reinterpret_cast<uint32_t*>(out);
    const uint32_t cb = f.cb;
    for (int b = b0; b < (WIDE ? min(B, b0 + 32) : B); ++b) {
      const uint32_t n = __shfl_sync(0xFFFFFFFFu, bcnt, b - b0);
      if (n == 0) continue;
      const uint32_t rs = __shfl_sync(0xFFFFFFFFu, brs, b - b0);
      const uint32_t p0 = __shfl_sync(0xFFFFFFFFu, bpre, b - b0);
      int32_t rprev = __shfl_sync(0xFFFFFFFFu, bprev, b - b0);
      const PackPar p = par[b];
      const uint32_t lv_ = (1u << p.q) - 1u;
      const uint32_t Rc = (uint32_t)p.bc + p0 * cb, Rq = (uint32_t)p.bq + p0 * p.q;
      const uint32_t Ec = Rc + n * cb, Eq = Rq + n * p.q;
      Carry cyc{0xFFFFFFFFu, 0u}, cyq{0xFFFFFFFFu, 0u};
      uint2 enext = lane < n ? __ldcs(gm + rs + lane) : make_uint2(0, 0);
      for (uint32_t j0 = 0; j0 < n; j0 += 32) {
        const uint32_t j = j0 + lane;
        const uint32_t nv = min(32u, n - j0);
        const bool valid = j < n;
        const uint2 e = enext;  // prefetched; the next window's entry is requested now
        if (j0 + 32 < n) enext = j + 32 < n ? __ldcs(gm + rs + j + 32) : make_uint2(0, 0);
        const uint32_t key = e.x & 0x7FFFFFFFu;
        const uint32_t x = e.y;
        const uint32_t code = (valid && !p.degen) ? quant_code(key, p.vmin, p.o64, p.inv, lv_) : 0u;
        const uint32_t row = fk.div(x);
        const uint32_t col = x - row * f.K;
        const int32_t rup = __shfl_up_sync(0xFFFFFFFFu, (int32_t)row, 1);
        const int32_t rp = lane ? rup : rprev;
        if (valid)
          for (int32_t r = rp + 1; r <= (int32_t)row; ++r) st_u32_le(out, p.rp + 4ull * (uint32_t)r, p0 + j);
        rprev = __shfl_sync(0xFFFFFFFFu, (int32_t)row, (int)nv - 1);
        // 8-bit fields are whole bytes of the MSB-first stream (bitstream.py:12-20): plain
        // byte stores, no word assembly (sections start on byte boundaries)
        if (cb == 8) { if (valid) out[(Rc >> 3) + j] = (uint8_t)col; }
        else pack_window(out32, pbuf[w][0], col, valid, cb, Rc, Ec, j0, nv, cyc);
        if (p.q == 8) { if (valid) out[(Rq >> 3) + j] = (uint8_t)code; }
        else pack_window(out32, pbuf[w][1], code, valid, p.q, Rq, Eq, j0, nv, cyq);
      }
    }
    }
  }
}

// ---------------------------------------------------------------------------------------
// K8: CRC-32 over bytes [4, P-4) (codec.py:316).  The range is cut into 2 KiB pieces
// aligned to its end; one warp computes a piece's raw CRC (crc_piece_warp), shifts it over
// the pieces after it with one multiply (kPieceShift) and XORs it into the IF's
// accumulator (GF(2) linearity).  Piece slots are sized from the capacity; the warp that
// completes an IF's last slot writes the CRC, the length and the status.
__global__ void __launch_bounds__(CNT, 6) enc_crc(EArgs a) {
  __shared__ uint32_t t4[1024];
  __shared__ uint32_t stage[CNT / 32][544];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < 1024; k += CNT) t4[k] = (&kCrcTab4[0][0])[k];
  __syncthreads();
  // each warp takes a contiguous range of the pieces (IFs walked forward, no per-piece search)
  const uint64_t GW = (uint64_t)gridDim.x * (CNT / 32), gw = (uint64_t)blockIdx.x * (CNT / 32) + w;
  const uint64_t total = a.seg_base[a.n];
  const uint64_t p0 = total * gw / GW, p1 = total * (gw + 1) / GW;
  PieceWalk pw;
  pw.init(a.seg_base, a.n);
  for (uint64_t gp = p0; gp < p1; ++gp) {
    const int ifi = pw.at(gp);
    const uint32_t piece = (uint32_t)(gp - pw.b0);
    const uint32_t npieces = pw.b1 - pw.b0;
    const IfInfo& f = a.info[ifi];
    IfSt& st = a.st[ifi];
    const uint32_t err = st.err;
    uint32_t part = 0;
    if (!err) {
      const uint64_t b0 = 4, b1 = st.P - 4;
      const uint64_t e1 = (uint64_t)piece * CRC_PIECE < b1 - b0 ? b1 - (uint64_t)piece * CRC_PIECE : b0;
      const uint64_t e0 = e1 - b0 > CRC_PIECE ? e1 - CRC_PIECE : b0;
      if (e0 < e1) {
        const uint32_t raw = crc_piece_warp(f.out, e0, e1, t4, stage[w]);
        part = raw ? crc_mult(kPieceShift[piece], raw) : 0u;
      }
    }
    if (lane == 0) {
      if (part) atomicXor(&st.crc_acc, part);
      __threadfence();
      if (atomicAdd(&st.seg_done, 1u) + 1 == npieces) {
        __threadfence();
        if (err == E_NONFINITE) { a.status[ifi] = SIF_ERR_NONFINITE; a.out_len[ifi] = 0; }
        else if (err) { a.status[ifi] = SIF_ERR_CAPACITY; a.out_len[ifi] = st.P; }
        else {
          const uint64_t P = st.P;
          st_u32_le_bytes(f.out, P - 4, crc_finish(atomicXor(&st.crc_acc, 0u), P - 8));
          a.out_len[ifi] = P;
          a.status[ifi] = SIF_OK;
        }
      }
    }
    __syncwarp();
  }
}

}  // namespace sif
