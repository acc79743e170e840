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
constexpr int CNT = 256;           // threads of chunk kernels
constexpr int DSH = 19;            // digit = |x| key >> 19 (12 bits)
constexpr int ND = 4096;           // digits per sign
constexpr int MAXB = 32;           // max blocks (M+ + M-) per IF
constexpr int SNT = 512;           // threads of the per-IF select kernel
constexpr int HB = 2048;           // radix histogram bins inside select_exact
constexpr int GCAP = 1024;         // in-SMEM exact ranking capacity
constexpr int GSM = 4096;          // gather list entries held in SMEM (K3)
constexpr uint32_t kInfKey = 0xFFFFFFFFu;

enum : uint32_t {
  F_KEEP_NONE = 1u, F_ONLY_NONZERO = 2u, F_ZERO_MODE = 4u, F_USE_CLS = 8u, F_TIE_ALL = 16u
};
enum : uint32_t { E_NONE = 0u, E_NONFINITE = 1u, E_CAPACITY = 2u };

// Static per-IF description, built on the host (sif_enc_upload).
struct IfInfo {
  const void* x;
  uint8_t* out;
  uint64_t cap, seed, T, kk;
  uint32_t N, K, cb, dtype;
  uint32_t ch0, nch;
  int32_t hslot;
  uint32_t pad;
  uint64_t list_off;  // workspace byte offset: vals u32[T], then idx u32[T]
  uint64_t gat_off;   // gather spill: vals u32[T], then idx u32[T]
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
};

struct EArgs {
  const IfInfo* info;
  IfSt* st;
  int n, nch, maxb, atkf_only;
  const uint32_t* ch_if;
  const uint32_t* ch_e0;
  uint32_t* ch_off;
  uint32_t* ch_cnt;
  uint32_t* ch_bcnt;   // [nch][maxb]
  uint32_t* ch_bpre;   // [nch][maxb]
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
};

__device__ __forceinline__ uint32_t* lv(const EArgs& a, const IfInfo& f) {
  return reinterpret_cast<uint32_t*>(a.ws + f.list_off);
}
__device__ __forceinline__ uint32_t* li(const EArgs& a, const IfInfo& f) {
  return reinterpret_cast<uint32_t*>(a.ws + f.list_off) + f.T;
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

__device__ __forceinline__ uint32_t warp_incl_scan_u32(uint32_t x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// ---------------------------------------------------------------------------------------
// List of (float bits, flat index) pairs: SMEM up to `cap` entries, global beyond.
struct List {
  uint32_t* sb;
  uint32_t* si;
  uint32_t* gb;
  uint32_t* gi;
  uint32_t cap;
  __device__ __forceinline__ uint32_t bits(uint32_t i) const { return i < cap ? sb[i] : __ldcg(gb + (i - cap)); }
  __device__ __forceinline__ uint32_t idx(uint32_t i) const { return i < cap ? si[i] : __ldcg(gi + (i - cap)); }
  __device__ __forceinline__ void set(uint32_t i, uint32_t b, uint32_t x) const {
    if (i < cap) { sb[i] = b; si[i] = x; }
    else { __stcg(gb + (i - cap), b); __stcg(gi + (i - cap), x); }
  }
};

// Visit every list element (order-free).  Global parts are read 4 elements per thread per
// step with independent loads.
template <int NT, class F>
__device__ __forceinline__ void list_foreach(const List& L, uint32_t n, F f) {
  const uint32_t ns = n < L.cap ? n : L.cap;
  for (uint32_t i = threadIdx.x; i < ns; i += NT) f(L.sb[i], L.si[i]);
  if (n > L.cap) {
    const uint32_t m = n - L.cap;
    for (uint32_t i0 = 0; i0 < m; i0 += 4 * NT) {
      uint32_t b[4], x[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t i = i0 + threadIdx.x + k * NT;
        b[k] = i < m ? __ldcg(L.gb + i) : 0u;
        x[k] = i < m ? __ldcg(L.gi + i) : 0u;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (i0 + threadIdx.x + k * NT < m) f(b[k], x[k]);
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
  uint32_t red[40];
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

// Multi-level radix select on 64-bit keys ("r-th largest") over list elements accepted by
// fn(bits, idx, &key).  Used for huge single-value tie sets.
template <int NT, class KeyFn>
__device__ uint64_t radix_select64(SelSh& sh, uint32_t* hist, const List& L, uint32_t n, uint64_t r, KeyFn fn) {
  const int shifts[6] = {53, 42, 31, 20, 9, 0};
  const int widths[6] = {11, 11, 11, 11, 11, 9};
  uint64_t prefix = 0, mask = 0;
  for (int lev = 0; lev < 6; ++lev) {
    const int shf = shifts[lev], nb = 1 << widths[lev];
    for (int i = threadIdx.x; i < nb; i += NT) hist[i] = 0;
    __syncthreads();
    list_foreach<NT>(L, n, [&](uint32_t b, uint32_t x) {
      uint64_t k;
      if (fn(b, x, k) && (k & mask) == prefix) atomicAdd(&hist[(int)((k >> shf) & (uint64_t)(nb - 1))], 1u);
    });
    __syncthreads();
    find_digit<NT>(sh, hist, nb, r);
    prefix |= (uint64_t)sh.fd_digit << shf;
    mask |= (uint64_t)(nb - 1) << shf;
    r -= sh.fd_above;
    __syncthreads();
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
template <int NT, class Pred, class KeyF, class SecF>
__device__ SelRes select_exact(SelSh& sh, uint32_t* scratch, const List& L, uint32_t n, Pred pred, KeyF keyf,
                               SecF secf, uint64_t klo, uint64_t khi, uint64_t r) {
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
    list_foreach<NT>(L, n, [&](uint32_t b, uint32_t x) {
      if (pred(b, x)) {
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
    res.sec = 0;
    if (!res.all_ties) {
      const uint32_t kk = (uint32_t)klo;
      const uint64_t top = radix_select64<NT>(sh, hist, L, n, r, [&](uint32_t b, uint32_t x, uint64_t& k) {
        if (!pred(b, x) || keyf(b) != kk) return false;
        k = ~secf(b, x);
        return true;
      });
      res.sec = ~top;
    }
    return res;
  }
  if (tid == 0) sh.gcount = 0;
  __syncthreads();
  list_foreach<NT>(L, n, [&](uint32_t b, uint32_t x) {
    if (pred(b, x)) {
      const uint64_t k = keyf(b);
      if (k >= klo && k < khi) {
        const uint32_t p = atomicAdd(&sh.gcount, 1u);
        gl[p].key = (uint32_t)k;
        gl[p].idx = x;
        gl[p].sec = secf(b, x);
      }
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
  if ((tid & 31) == 0) { sh.red[tid >> 5] = gt; sh.red[16 + (tid >> 5)] = eq; }
  __syncthreads();
  uint64_t tgt = 0, teq = 0;
  for (int w = 0; w < NW; ++w) { tgt += sh.red[w]; teq += sh.red[16 + w]; }
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
// Stream one chunk (n <= CH elements starting at flat index e0): candidates (|x| >= lo for
// x >= 0, |x| >= lo_neg for x < 0) are staged per warp in flat order at sv/si[w*EW ...),
// wcnt[w] = count.  Warp w owns elements [w*EW, (w+1)*EW) of the chunk; each lane loads V
// consecutive elements per step (one 128-bit load).  hist (if non-null): per-sign digit
// counts of the candidates.  Per-thread outputs: max |x| key, count of |x| >= lo, digit range.
template <int DT, int NT>
__device__ __forceinline__ void stream_chunk(const void* x, uint32_t e0, uint32_t n, uint32_t lo, uint32_t lo_neg,
                                             uint32_t* sv, uint32_t* si, uint32_t* hist, uint32_t* wcnt,
                                             uint32_t& mk, uint32_t& clo, uint32_t& dmin, uint32_t& dmax) {
  constexpr int NW = NT / 32;
  constexpr int EW = CH / NW;
  constexpr int V = DT == SIF_DTYPE_F32 ? 4 : 8;
  constexpr int IT = EW / (32 * V);
  static_assert(IT >= 1, "chunk too small for the CTA");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t wb = (uint32_t)w * EW;
  uint32_t v[IT][V];
  const bool full = wb + EW <= n;
#pragma unroll
  for (int j = 0; j < IT; ++j) {
    const uint32_t o = wb + (uint32_t)j * 32u * V + (uint32_t)lane * V;
    if (full) {
      if (DT == SIF_DTYPE_F32) {
        const uint4 q = __ldcs(reinterpret_cast<const uint4*>(reinterpret_cast<const uint32_t*>(x) + e0 + o));
        v[j][0] = q.x; v[j][1] = q.y; v[j][2] = q.z; v[j][3] = q.w;
      } else {
        const uint4 q = __ldcs(reinterpret_cast<const uint4*>(reinterpret_cast<const unsigned short*>(x) + e0 + o));
        const uint32_t ww[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) { v[j][2 * k] = ww[k] << 16; v[j][2 * k + 1] = ww[k] & 0xFFFF0000u; }
      }
    } else {
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const uint32_t e = o + k;
        uint32_t b = 0;
        if (e < n) {
          if (DT == SIF_DTYPE_F32) b = __ldcs(reinterpret_cast<const uint32_t*>(x) + e0 + e);
          else b = (uint32_t)__ldcs(reinterpret_cast<const unsigned short*>(x) + e0 + e) << 16;
        }
        v[j][k] = b;
      }
    }
  }
  uint32_t run = 0;
  const uint32_t lt = (1u << lane) - 1u;
  (void)lt;
#pragma unroll
  for (int j = 0; j < IT; ++j) {
    const uint32_t o = wb + (uint32_t)j * 32u * V + (uint32_t)lane * V;
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const uint32_t b = v[j][k];
      const uint32_t key = b & 0x7FFFFFFFu;
      const bool in = full || (o + k < n);
      mk = max(mk, in ? key : 0u);
      const uint32_t thr = (b >> 31) ? lo_neg : lo;
      const bool c = in && key >= thr;
      clo += (in && key >= lo) ? 1u : 0u;
      m |= c ? (1u << k) : 0u;
    }
    const uint32_t cnt = __popc(m);
    const uint32_t incl = warp_incl_scan_u32(cnt);
    uint32_t pos = wb + run + incl - cnt;
    run += __shfl_sync(0xFFFFFFFFu, incl, 31);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      if ((m >> k) & 1u) {
        const uint32_t b = v[j][k];
        sv[pos] = b;
        si[pos] = e0 + o + k;
        ++pos;
        if (hist) {
          const uint32_t d = (b & 0x7FFFFFFFu) >> DSH;
          atomicAdd(&hist[((b >> 31) ? ND : 0) + d], 1u);
          dmin = min(dmin, d);
          dmax = max(dmax, d);
        }
      }
    }
  }
  if (lane == 0) wcnt[w] = run;
}

// ---------------------------------------------------------------------------------------
// K1: per-IF setup: accumulators and the sampled bracket lo (speculation only: a missed
// bracket is detected in K3 and the IF re-streamed).
__global__ void __launch_bounds__(256) enc_prep(EArgs a) {
  constexpr int NT = 256;
  __shared__ uint32_t sh8k[8192];
  __shared__ SelSh sh;
  const int i = blockIdx.x, tid = threadIdx.x;
  const IfInfo f = a.info[i];
  IfSt& st = a.st[i];
  for (int b = tid; b < a.maxb; b += NT) { st.bmin[b] = 0x7FFFFFFFu; st.bmax[b] = 0u; }
  for (int k = tid; k < a.maxb * 16; k += NT) st.S[k] = 0ull;
  if (f.hslot >= 0) {
    uint4* h = reinterpret_cast<uint4*>(a.hist + (uint64_t)f.hslot * 2 * ND);
    for (int k = tid; k < 2 * ND / 4; k += NT) h[k] = make_uint4(0, 0, 0, 0);
  }
  const uint64_t T = f.T, kk = f.kk;
  uint32_t lo = 1;
  if (T > 32768 && kk > 0 && 2 * kk <= T) {
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
  }
  uint32_t lo_neg = lo;
  if (a.lam > 0.0 && lo > 1) {
    const double t = __dmul_rn(__dsub_rn(1.0, a.lam), (double)__uint_as_float(lo));
    const uint32_t k2 = __float_as_uint(__double2float_rd(t));
    lo_neg = k2 > 1 ? k2 : 1u;
  }
  if (tid == 0) {
    st.lo = lo; st.lo_neg = lo_neg; st.ncand = 0; st.maxkey = 0; st.cnt_lo = 0; st.err = E_NONE; st.flags = 0;
    st.P = 0;
  }
}

// ---------------------------------------------------------------------------------------
// K2: stream chunks (persistent CTAs).
template <int NT>
__device__ __forceinline__ void stream_and_emit(const EArgs& a, uint32_t c, const IfInfo& f, uint32_t lo,
                                                uint32_t lo_neg, uint32_t* sv, uint32_t* si, uint32_t* hist,
                                                uint32_t* wcnt, uint32_t* misc, uint32_t* list_cursor,
                                                bool global_reserve, IfSt* st) {
  constexpr int NW = NT / 32;
  constexpr int EW = CH / NW;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t e0 = a.ch_e0[c];
  const uint32_t n = (uint32_t)min((uint64_t)CH, f.T - e0);
  uint32_t mk = 0, clo = 0, dmin = 0xFFFFFFFFu, dmax = 0;
  if (f.dtype == SIF_DTYPE_BF16)
    stream_chunk<SIF_DTYPE_BF16, NT>(f.x, e0, n, lo, lo_neg, sv, si, hist, wcnt, mk, clo, dmin, dmax);
  else
    stream_chunk<SIF_DTYPE_F32, NT>(f.x, e0, n, lo, lo_neg, sv, si, hist, wcnt, mk, clo, dmin, dmax);
  mk = __reduce_max_sync(0xFFFFFFFFu, mk);
  clo = __reduce_add_sync(0xFFFFFFFFu, clo);
  dmin = __reduce_min_sync(0xFFFFFFFFu, dmin);
  dmax = __reduce_max_sync(0xFFFFFFFFu, dmax);
  if (lane == 0) {
    atomicMax(&misc[0], mk);
    atomicAdd(&misc[1], clo);
    atomicMin(&misc[2], dmin);
    atomicMax(&misc[3], dmax);
  }
  __syncthreads();
  if (tid == 0) {
    uint32_t acc = 0;
    for (int k = 0; k < NW; ++k) { const uint32_t t = wcnt[k]; wcnt[NW + k] = acc; acc += t; }
    uint32_t off;
    if (global_reserve) {
      off = atomicAdd(&st->ncand, acc);
      atomicMax(&st->maxkey, misc[0]);
      atomicAdd(&st->cnt_lo, misc[1]);
    } else {
      off = *list_cursor;
      *list_cursor = off + acc;
    }
    a.ch_off[c] = off;
    a.ch_cnt[c] = acc;
    misc[4] = off;
  }
  __syncthreads();
  {
    uint32_t* gv = lv(a, f);
    uint32_t* gi = li(a, f);
    const uint32_t base = misc[4] + wcnt[NW + w];
    const uint32_t m = wcnt[w];
    for (uint32_t k = lane; k < m; k += 32) {
      gv[base + k] = sv[w * EW + k];
      gi[base + k] = si[w * EW + k];
    }
  }
  if (hist && global_reserve && misc[2] <= misc[3]) {
    uint32_t* gh = a.hist + (uint64_t)f.hslot * 2 * ND;
    const uint32_t d0 = misc[2], nr = misc[3] - misc[2] + 1;
    for (uint32_t k = tid; k < 2 * nr; k += NT) {
      const uint32_t d = (k < nr ? 0u : (uint32_t)ND) + d0 + (k < nr ? k : k - nr);
      const uint32_t h = hist[d];
      if (h) { atomicAdd(gh + d, h); hist[d] = 0; }
    }
  }
  __syncthreads();
  if (tid == 0) { misc[0] = 0; misc[1] = 0; misc[2] = 0xFFFFFFFFu; misc[3] = 0; }
  __syncthreads();
}

__global__ void __launch_bounds__(CNT) enc_stream(EArgs a) {
  extern __shared__ __align__(16) uint8_t dsm_raw[];
  uint32_t* dsm = reinterpret_cast<uint32_t*>(dsm_raw);
  __shared__ uint32_t wcnt[2 * (CNT / 32)];
  __shared__ uint32_t misc[8];
  uint32_t* sv = dsm;
  uint32_t* si = dsm + CH;
  uint32_t* hist = dsm + 2 * CH;
  for (int k = threadIdx.x; k < 2 * ND; k += CNT) hist[k] = 0;
  if (threadIdx.x == 0) { misc[0] = 0; misc[1] = 0; misc[2] = 0xFFFFFFFFu; misc[3] = 0; }
  __syncthreads();
  for (uint32_t c = blockIdx.x; c < (uint32_t)a.nch; c += gridDim.x) {
    const uint32_t ifi = a.ch_if[c];
    const IfInfo f = a.info[ifi];
    IfSt* st = a.st + ifi;
    const uint32_t lo = st->lo, lo_neg = st->lo_neg;
    stream_and_emit<CNT>(a, c, f, lo, lo_neg, sv, si, f.hslot >= 0 ? hist : nullptr, wcnt, misc, nullptr, true, st);
  }
}

// ---------------------------------------------------------------------------------------
// K3: per-IF selection.
struct K3Sh {
  SelSh s;
  uint32_t wcnt[2 * (SNT / 32)];
  uint32_t misc[8];
  uint32_t cursor;
  uint32_t nA, nB;
  uint32_t keptA[2];
  uint64_t cnt_nz;
  uint32_t pend_n;
  uint32_t pend_s[MAXB], pend_d[MAXB], pend_r[MAXB], pend_ci[MAXB];
};

__global__ void __launch_bounds__(SNT) enc_select(EArgs a) {
  constexpr int NT = SNT;
  extern __shared__ __align__(16) uint8_t dsm_raw[];
  uint32_t* dsm = reinterpret_cast<uint32_t*>(dsm_raw);
  __shared__ K3Sh k3;
  SelSh& sh = k3.s;
  uint32_t* hist = dsm;                         // 2*ND
  uint32_t* scratch = dsm + 2 * ND;             // 2*HB + GCAP*4
  uint32_t* gbuf = scratch + 2 * HB + GCAP * 4; // 2*GSM (also the re-stream stage)
  const int ifi = blockIdx.x, tid = threadIdx.x;
  const IfInfo f = a.info[ifi];
  IfSt& st = a.st[ifi];
  const uint64_t kk = f.kk, seed = f.seed;
  if (st.maxkey >= kNonFiniteKey) {
    if (tid == 0) {
      st.err = E_NONFINITE;
      if (a.atkf_only) a.status[ifi] = SIF_ERR_NONFINITE;
    }
    return;
  }
  uint32_t lo = st.lo, lo_neg = st.lo_neg;
  const uint32_t floor_lo = a.atkf_only ? 0u : 1u;
  uint32_t ncand = st.ncand;
  bool hist_ok = false;
  if (kk > 0 && st.cnt_lo < kk && lo > floor_lo) {
    // bracket missed (or tau == 0): re-stream keeping every nonzero (every element in
    // ATKF-only mode); this CTA writes the list in chunk order and the histogram in SMEM
    lo = floor_lo;
    lo_neg = floor_lo;
    for (int k = tid; k < 2 * ND; k += NT) hist[k] = 0;
    if (tid == 0) { k3.cursor = 0; k3.misc[0] = 0; k3.misc[1] = 0; k3.misc[2] = 0xFFFFFFFFu; k3.misc[3] = 0; }
    __syncthreads();
    for (uint32_t c = f.ch0; c < f.ch0 + f.nch; ++c)
      stream_and_emit<NT>(a, c, f, lo, lo_neg, gbuf, gbuf + CH, hist, k3.wcnt, k3.misc, &k3.cursor, false, &st);
    ncand = k3.cursor;
    hist_ok = true;
  } else if (f.hslot >= 0) {
    const uint4* gh = reinterpret_cast<const uint4*>(a.hist + (uint64_t)f.hslot * 2 * ND);
    uint4* h4 = reinterpret_cast<uint4*>(hist);
    for (int k = tid; k < 2 * ND / 4; k += NT) h4[k] = __ldcg(gh + k);
    hist_ok = true;
  }
  const List L{nullptr, nullptr, lv(a, f), li(a, f), 0};
  if (!hist_ok) {
    for (int k = tid; k < 2 * ND; k += NT) hist[k] = 0;
    __syncthreads();
    list_foreach<NT>(L, ncand, [&](uint32_t b, uint32_t) {
      atomicAdd(&hist[((b >> 31) ? ND : 0) + ((b & 0x7FFFFFFFu) >> DSH)], 1u);
    });
  }
  __syncthreads();
  // candidates with key != 0 (only lo == 0 admits zeros)
  uint64_t cnt_nz = ncand;
  if (lo == 0) {
    cnt_nz = (uint64_t)ncand - hist[0] - hist[ND];  // digit 0 holds zeros and tiny values
    uint32_t tiny = 0;
    list_foreach<NT>(L, ncand, [&](uint32_t b, uint32_t) {
      const uint32_t key = b & 0x7FFFFFFFu;
      tiny += (key != 0 && (key >> DSH) == 0) ? 1u : 0u;
    });
    tiny = __reduce_add_sync(0xFFFFFFFFu, tiny);
    if (tid == 0) k3.cnt_nz = 0;
    __syncthreads();
    if ((tid & 31) == 0) atomicAdd((unsigned long long*)&k3.cnt_nz, (unsigned long long)tiny);
    __syncthreads();
    cnt_nz += k3.cnt_nz;
    __syncthreads();
  }
  const bool zero_mode = kk > 0 && lo == 0;
  const bool keep_none = kk == 0;
  const bool only_nonzero = kk > 0 && cnt_nz < kk && !zero_mode;
  auto hash_of = [seed](uint32_t, uint32_t x) -> uint64_t { return splitmix(seed, x); };
  auto key31 = [](uint32_t b) -> uint64_t { return b & 0x7FFFFFFFu; };
  auto all_pred = [](uint32_t, uint32_t) { return true; };
  uint32_t tau_key = 0;
  uint64_t ck_star = 0, h_star = 0;
  bool tie_all = true;
  int dtau = -1;  // digit of tau on the fast path (-1: every candidate bin counts fully)
  const bool use_cls = a.lam > 0.0 && kk > 0 && !only_nonzero;
  const bool fast = !zero_mode && !use_cls;
  List A{gbuf, gbuf + GSM, reinterpret_cast<uint32_t*>(a.ws + f.gat_off),
         reinterpret_cast<uint32_t*>(a.ws + f.gat_off) + f.T, GSM};
  uint32_t nA = 0;
  if (kk > 0 && !only_nonzero) {
    if (zero_mode && cnt_nz < kk) {
      // tau == 0 (ATKF-only mode): every nonzero is kept; choose kk - nnz zeros by hash
      const SelRes s = select_exact<NT>(sh, scratch, L, ncand, all_pred, key31, hash_of, 0, 1, kk - cnt_nz);
      h_star = s.sec;
      tie_all = s.all_ties;
    } else if (!fast) {
      const uint64_t klo = lo_neg < lo ? lo_neg : lo;
      const SelRes s = select_exact<NT>(sh, scratch, L, ncand, all_pred, key31, hash_of, klo,
                                        (uint64_t)st.maxkey + 1, kk);
      tau_key = s.key;
      ck_star = s.key;
      h_star = s.sec;
      tie_all = s.all_ties;
    } else {
      // digit of tau over both signs, then the bin's elements -> exact select
      uint32_t* comb = scratch;
      for (int k = tid; k < ND; k += NT) comb[k] = hist[k] + hist[ND + k];
      __syncthreads();
      find_digit<NT>(sh, comb, ND, kk);
      dtau = (int)sh.fd_digit;
      const uint64_t rt = kk - sh.fd_above;
      if (tid == 0) k3.nA = 0;
      __syncthreads();
      list_foreach<NT>(L, ncand, [&](uint32_t b, uint32_t x) {
        if (((b & 0x7FFFFFFFu) >> DSH) == (uint32_t)dtau) {
          const uint32_t p = atomicAdd(&k3.nA, 1u);
          A.set(p, b, x);
        }
      });
      __syncthreads();
      nA = k3.nA;
      const SelRes s = select_exact<NT>(sh, scratch, A, nA, all_pred, key31, hash_of, (uint64_t)dtau << DSH,
                                        (uint64_t)(dtau + 1) << DSH, rt);
      tau_key = s.key;
      ck_star = s.key;
      h_star = s.sec;
      tie_all = s.all_ties;
    }
  }
  const double tau = kk > 0 ? (double)__uint_as_float(tau_key) : (double)__uint_as_float(st.maxkey);
  const double tau_p = __dmul_rn(__dadd_rn(1.0, a.lam), tau);
  const double tau_m = -__dmul_rn(__dsub_rn(1.0, a.lam), tau);
  if (use_cls) {
    auto ckey = [tau_p, tau_m](uint32_t b) -> uint64_t {
      const double v = (double)__uint_as_float(b);
      return ((v > tau_p || v < tau_m) ? (1ull << 31) : 0ull) | (uint64_t)(b & 0x7FFFFFFFu);
    };
    const SelRes s = select_exact<NT>(sh, scratch, L, ncand, all_pred, ckey, hash_of, 0, 1ull << 32, kk);
    ck_star = s.key;
    h_star = s.sec;
    tie_all = s.all_ties;
  }
  auto kept_of = [&](uint32_t b, uint32_t x) -> bool {
    if (keep_none) return false;
    const uint32_t key = b & 0x7FFFFFFFu;
    if (only_nonzero) return key != 0;
    if (!zero_mode && key == 0) return false;
    uint64_t ck = key;
    if (use_cls) {
      const double v = (double)__uint_as_float(b);
      if (v > tau_p || v < tau_m) ck |= 1ull << 31;
    }
    if (ck != ck_star) return ck > ck_star;
    return tie_all || splitmix(seed, x) <= h_star;
  };
  // ---- ATKF-only: kept flat indices in ascending order, tau
  if (a.atkf_only) {
    int64_t* out = a.kept_out + a.kept_off[ifi];
    uint64_t run = 0;
    for (uint32_t c = f.ch0; c < f.ch0 + f.nch; ++c) {
      const uint32_t off = a.ch_off[c], cn = a.ch_cnt[c];
      for (uint32_t base = 0; base < cn; base += NT) {
        const uint32_t j = base + tid;
        bool kp = false;
        uint32_t x = 0;
        if (j < cn) {
          x = __ldcg(L.gi + off + j);
          kp = kept_of(__ldcg(L.gb + off + j), x);
        }
        uint32_t tot;
        const uint32_t ex = block_excl_scan_u32(kp ? 1u : 0u, sh.red, &tot);
        if (kp) out[run + ex] = (int64_t)x;
        run += tot;
      }
    }
    if (tid == 0) {
      a.tau3[3 * ifi + 0] = tau;
      a.tau3[3 * ifi + 1] = tau_p;
      a.tau3[3 * ifi + 2] = tau_m;
      a.status[ifi] = SIF_OK;
    }
    return;
  }
  // ---- kept nonzeros per sign
  uint64_t nnz[2] = {0, 0};
  if (fast) {
    if (tid < 2) k3.keptA[tid] = 0;
    __syncthreads();
    if (dtau >= 0) {
      uint32_t c0 = 0, c1 = 0;
      list_foreach<NT>(A, nA, [&](uint32_t b, uint32_t x) {
        if (kept_of(b, x)) { if (b >> 31) ++c1; else ++c0; }
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
    uint32_t c0 = 0, c1 = 0;
    list_foreach<NT>(L, ncand, [&](uint32_t b, uint32_t x) {
      if ((b & 0x7FFFFFFFu) != 0 && kept_of(b, x)) { if (b >> 31) ++c1; else ++c0; }
    });
    c0 = __reduce_add_sync(0xFFFFFFFFu, c0);
    c1 = __reduce_add_sync(0xFFFFFFFFu, c1);
    if (tid < 2) k3.s.cnt[tid] = 0;
    __syncthreads();
    if ((tid & 31) == 0) { atomicAdd(&k3.s.cnt[0], c0); atomicAdd(&k3.s.cnt[1], c1); }
    __syncthreads();
    nnz[0] = k3.s.cnt[0];
    nnz[1] = k3.s.cnt[1];
    __syncthreads();
  }
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
  if (fast) {
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
      if ((int)dc == dtau) {
        const SelRes r = select_exact<NT>(
            sh, scratch, A, nA, [&](uint32_t b, uint32_t x) { return (b >> 31) == s && kept_of(b, x); }, key31,
            [](uint32_t, uint32_t x) -> uint64_t { return x; }, (uint64_t)dc << DSH, (uint64_t)(dc + 1) << DSH, rc);
        if (tid == 0) { st.cut_key[ci] = r.key; st.cut_idx[ci] = (uint32_t)r.sec; }
      } else if (tid == 0) {
        const uint32_t p = k3.pend_n++;
        k3.pend_s[p] = s; k3.pend_d[p] = dc; k3.pend_r[p] = (uint32_t)rc; k3.pend_ci[p] = (uint32_t)ci;
      }
      __syncthreads();
    }
    const uint32_t np = k3.pend_n;
    if (np > 0) {
      // gather every pending cut bin in one pass (B reuses A's storage)
      uint32_t* pm = scratch;  // bitmap of pending (sign, digit): 2*ND bits
      for (int k = tid; k < 2 * ND / 32; k += NT) pm[k] = 0;
      __syncthreads();
      if (tid < (int)np) {
        const uint32_t d = k3.pend_s[tid] * ND + k3.pend_d[tid];
        atomicOr(&pm[d >> 5], 1u << (d & 31));
      }
      if (tid == 0) k3.nB = 0;
      __syncthreads();
      List Bl = A;
      list_foreach<NT>(L, ncand, [&](uint32_t b, uint32_t x) {
        const uint32_t d = ((b >> 31) ? ND : 0) + ((b & 0x7FFFFFFFu) >> DSH);
        if ((pm[d >> 5] >> (d & 31)) & 1u) {
          const uint32_t p = atomicAdd(&k3.nB, 1u);
          Bl.set(p, b, x);
        }
      });
      __syncthreads();
      const uint32_t nB = k3.nB;
      for (uint32_t p = 0; p < np; ++p) {
        const uint32_t s = k3.pend_s[p], dc = k3.pend_d[p];
        const SelRes r = select_exact<NT>(
            sh, scratch, Bl, nB,
            [&](uint32_t b, uint32_t) { return (b >> 31) == s && ((b & 0x7FFFFFFFu) >> DSH) == dc; }, key31,
            [](uint32_t, uint32_t x) -> uint64_t { return x; }, (uint64_t)dc << DSH, (uint64_t)(dc + 1) << DSH,
            k3.pend_r[p]);
        if (tid == 0) { st.cut_key[k3.pend_ci[p]] = r.key; st.cut_idx[k3.pend_ci[p]] = (uint32_t)r.sec; }
        __syncthreads();
      }
    }
  } else {
    for (int ci = 0; ci < ncut; ++ci) {
      const uint32_t s = ci < ncut0 ? 0u : 1u;
      const int j = (s == 0 ? ci : ci - ncut0) + 1;
      const uint64_t rank0 = (uint64_t)j * base[s];
      const SelRes r = select_exact<NT>(
          sh, scratch, L, ncand,
          [&](uint32_t b, uint32_t x) { return (b >> 31) == s && (b & 0x7FFFFFFFu) != 0 && kept_of(b, x); }, key31,
          [](uint32_t, uint32_t x) -> uint64_t { return x; }, 1, 1ull << 31, rank0 + 1);
      if (tid == 0) { st.cut_key[ci] = r.key; st.cut_idx[ci] = (uint32_t)r.sec; }
      __syncthreads();
    }
  }
  if (tid == 0) {
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
// K4: kept test, block ids, stable regroup of each chunk segment by block.
struct K4Sh {
  KeptCtx kc;
  uint32_t cur_if;
  uint32_t wcnt[CNT / 32][MAXB];
  uint32_t wmin[CNT / 32][MAXB];
  uint32_t wmax[CNT / 32][MAXB];
  uint32_t wlast[CNT / 32][MAXB];
  uint32_t wpos[CNT / 32][MAXB];
  uint32_t bstart[MAXB];
};

__global__ void __launch_bounds__(CNT) enc_members(EArgs a) {
  constexpr int NW = CNT / 32;
  extern __shared__ __align__(16) uint8_t dsm_raw[];
  uint32_t* dsm = reinterpret_cast<uint32_t*>(dsm_raw);
  __shared__ K4Sh sh;
  uint32_t* iv = dsm;
  uint32_t* ix = dsm + CH;
  uint32_t* ov = dsm + 2 * CH;
  uint32_t* ox = dsm + 3 * CH;
  int8_t* bid = reinterpret_cast<int8_t*>(dsm + 4 * CH);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  if (tid == 0) sh.cur_if = 0xFFFFFFFFu;
  __syncthreads();
  for (uint32_t c = blockIdx.x; c < (uint32_t)a.nch; c += gridDim.x) {
    const uint32_t ifi = a.ch_if[c];
    const IfInfo& f = a.info[ifi];
    IfSt& st = a.st[ifi];
    if (st.err) continue;
    if (sh.cur_if != ifi) {
      __syncthreads();
      if (tid == 0) load_kept_ctx(sh.kc, st, f.seed);
      __syncthreads();
      if (tid == 0) sh.cur_if = ifi;
    }
    const int B = (int)st.B;
    const uint32_t off = a.ch_off[c], n = a.ch_cnt[c];
    const uint32_t K = f.K;
    uint32_t* gv = lv(a, f);
    uint32_t* gx = li(a, f);
    for (uint32_t k = tid; k < n; k += CNT) { iv[k] = __ldcg(gv + off + k); ix[k] = __ldcg(gx + off + k); }
    for (int k = tid; k < NW * MAXB; k += CNT) {
      (&sh.wcnt[0][0])[k] = 0; (&sh.wmin[0][0])[k] = 0x7FFFFFFFu; (&sh.wmax[0][0])[k] = 0; (&sh.wlast[0][0])[k] = 0;
    }
    __syncthreads();
    const uint32_t seg = (((n + NW - 1) / NW) + 31u) & ~31u;
    const uint32_t w0 = min(n, (uint32_t)w * seg), w1 = min(n, w0 + seg);
    // pass 1: block ids, per-warp counts, min/max keys, last member index per block
    for (uint32_t i = w0; i < w1; i += 32) {
      const uint32_t e = i + lane;
      int blk = -1;
      uint32_t key = 0, x = 0;
      if (e < w1) {
        const uint32_t b = iv[e];
        x = ix[e];
        key = b & 0x7FFFFFFFu;
        if (sh.kc.kept(b, x)) blk = sh.kc.block_of(b, x);
        bid[e] = (int8_t)blk;
      }
      uint32_t pend = __ballot_sync(0xFFFFFFFFu, blk >= 0);
      while (pend) {
        const int ld = __ffs(pend) - 1;
        const int bb = __shfl_sync(0xFFFFFFFFu, blk, ld);
        const uint32_t peers = __ballot_sync(0xFFFFFFFFu, blk == bb);
        const uint32_t mn = __reduce_min_sync(0xFFFFFFFFu, blk == bb ? key : 0x7FFFFFFFu);
        const uint32_t mx = __reduce_max_sync(0xFFFFFFFFu, blk == bb ? key : 0u);
        const uint32_t xl = __reduce_max_sync(0xFFFFFFFFu, blk == bb ? x + 1u : 0u);
        if (lane == 0) {
          sh.wcnt[w][bb] += __popc(peers);
          sh.wmin[w][bb] = min(sh.wmin[w][bb], mn);
          sh.wmax[w][bb] = max(sh.wmax[w][bb], mx);
          sh.wlast[w][bb] = max(sh.wlast[w][bb], xl);
        }
        pend &= ~peers;
      }
    }
    __syncthreads();
    // per-block totals and offsets (block runs in block order, warps in flat order)
    if (tid < B) {
      const int b = tid;
      uint32_t acc = 0, mn = 0x7FFFFFFFu, mx = 0, xl = 0;
      for (int k = 0; k < NW; ++k) {
        sh.wpos[k][b] = acc;
        acc += sh.wcnt[k][b];
        mn = min(mn, sh.wmin[k][b]);
        mx = max(mx, sh.wmax[k][b]);
        xl = max(xl, sh.wlast[k][b]);
      }
      sh.bstart[b] = acc;  // total (turned into start below)
      a.ch_bcnt[(uint64_t)c * a.maxb + b] = acc;
      a.ch_blast[(uint64_t)c * a.maxb + b] = xl ? (int32_t)((xl - 1u) / K) : -1;
      if (acc) { atomicMin(&st.bmin[b], mn); atomicMax(&st.bmax[b], mx); }
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t acc = 0;
      for (int b = 0; b < B; ++b) { const uint32_t t = sh.bstart[b]; sh.bstart[b] = acc; acc += t; }
    }
    __syncthreads();
    for (int k = tid; k < NW * B; k += CNT) {
      const int ww = k / B, b = k - ww * B;
      sh.wpos[ww][b] += sh.bstart[b];
    }
    __syncthreads();
    // pass 2: stable scatter into block runs
    for (uint32_t i = w0; i < w1; i += 32) {
      const uint32_t e = i + lane;
      const int blk = e < w1 ? (int)bid[e] : -1;
      const uint32_t peers = __match_any_sync(0xFFFFFFFFu, blk);
      if (blk >= 0) {
        const uint32_t dst = sh.wpos[w][blk] + __popc(peers & lt);
        ov[dst] = iv[e];
        ox[dst] = ix[e];
      }
      __syncwarp();
      if (blk >= 0 && lane == __ffs(peers) - 1) sh.wpos[w][blk] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    uint32_t tot = 0;
    for (int b = 0; b < B; ++b) tot += a.ch_bcnt[(uint64_t)c * a.maxb + b];
    for (uint32_t k = tid; k < tot; k += CNT) { __stcg(gv + off + k, ov[k]); __stcg(gx + off + k, ox[k]); }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------
// K5: ABQ distortion sums: S[b][q] = sum |code_qbit >> (qbit - q) - code_q| (quant.py:88-99)
struct K5Sh {
  uint32_t cur_if;
  double vmin[MAXB];
  double o[MAXB][17];
  double inv[MAXB][17];
  uint32_t act[MAXB];
  uint32_t red[CNT / 32][17];
};

__global__ void __launch_bounds__(CNT) enc_abq(EArgs a) {
  constexpr int NW = CNT / 32;
  __shared__ K5Sh sh;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int qb = a.q_bit;
  if (tid == 0) sh.cur_if = 0xFFFFFFFFu;
  __syncthreads();
  for (uint32_t c = blockIdx.x; c < (uint32_t)a.nch; c += gridDim.x) {
    const uint32_t ifi = a.ch_if[c];
    const IfInfo& f = a.info[ifi];
    IfSt& st = a.st[ifi];
    if (st.err) continue;
    const int B = (int)st.B;
    if (sh.cur_if != ifi) {
      __syncthreads();
      for (int k = tid; k < B * 16; k += CNT) {
        const int b = k >> 4, q = (k & 15) + 1;
        const uint32_t mn = st.bmin[b], mx = st.bmax[b];
        const double vmin = (double)__uint_as_float(mn), vmax = (double)__uint_as_float(mx);
        if (q <= qb) {
          const double o = __ddiv_rn(__dsub_rn(vmax, vmin), (double)((1u << q) - 1u));
          sh.o[b][q] = o;
          sh.inv[b][q] = __drcp_rn(o);
        }
        if (q == 1) { sh.vmin[b] = vmin; sh.act[b] = mn < mx ? 1u : 0u; }
      }
      __syncthreads();
      if (tid == 0) sh.cur_if = ifi;
    }
    const uint32_t off = a.ch_off[c];
    const uint32_t* gv = lv(a, f) + off;
    uint32_t rs = 0;
    for (int b = 0; b < B; ++b) {
      const uint32_t nb = a.ch_bcnt[(uint64_t)c * a.maxb + b];
      if (nb == 0 || !sh.act[b]) { rs += nb; continue; }
      uint32_t acc[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) acc[q] = 0;
      const double vmin = sh.vmin[b];
      const uint32_t lref = (1u << qb) - 1u;
      for (uint32_t k = tid; k < nb; k += CNT) {
        const uint32_t key = __ldcg(gv + rs + k) & 0x7FFFFFFFu;
        const uint32_t cr = quant_code(key, vmin, sh.o[b][qb], sh.inv[b][qb], lref);
#pragma unroll
        for (int q = 1; q < 16; ++q) {
          if (q < qb) {
            const uint32_t cq = quant_code(key, vmin, sh.o[b][q], sh.inv[b][q], (1u << q) - 1u);
            const uint32_t r = cr >> (qb - q);
            acc[q] += r > cq ? r - cq : cq - r;
          }
        }
      }
#pragma unroll
      for (int q = 1; q < 16; ++q) {
        if (q < qb) {
          const uint32_t v = __reduce_add_sync(0xFFFFFFFFu, acc[q]);
          if (lane == 0) sh.red[w][q] = v;
        }
      }
      __syncthreads();
      if (tid >= 1 && tid < qb) {
        uint64_t t = 0;
        for (int k = 0; k < NW; ++k) t += sh.red[k][tid];
        if (t) atomicAdd((unsigned long long*)&st.S[b * 16 + tid], (unsigned long long)t);
      }
      __syncthreads();
      rs += nb;
    }
  }
}

// ---------------------------------------------------------------------------------------
// K6: per-IF q*, layout, header, chunk prefixes, row_ptr tails.
__device__ __forceinline__ void st_u32_le(uint8_t* base, uint64_t off, uint32_t v) { st_u32_le_bytes(base, off, v); }

__global__ void __launch_bounds__(256) enc_layout(EArgs a) {
  constexpr int NT = 256;
  __shared__ uint32_t scan32[40];
  __shared__ uint64_t scan64[40];
  __shared__ uint64_t s_bn[MAXB];
  __shared__ int32_t s_last[MAXB];
  __shared__ uint32_t s_q[MAXB];
  __shared__ uint64_t s_P;
  const int ifi = blockIdx.x, tid = threadIdx.x;
  const IfInfo f = a.info[ifi];
  IfSt& st = a.st[ifi];
  if (st.err) return;
  const int B = (int)st.B;
  const uint32_t ch0 = f.ch0, nch = f.nch;
  // chunk prefixes per block: member offsets and the row of the previous member
  for (int b = 0; b < B; ++b) {
    uint32_t run = 0;
    int32_t lastp = -1;
    for (uint32_t t0 = 0; t0 < nch; t0 += NT) {
      const uint32_t k = t0 + tid;
      const uint64_t ci = (uint64_t)(ch0 + k) * a.maxb + b;
      const uint32_t v = k < nch ? a.ch_bcnt[ci] : 0u;
      const int32_t l = k < nch ? a.ch_blast[ci] : -1;
      uint32_t tot;
      const uint32_t ex = block_excl_scan_u32(v, scan32, &tot);
      // exclusive max-scan of last rows (rows grow with the chunk index)
      int32_t m = l;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xFFFFFFFFu, m, o);
        if ((tid & 31) >= o) m = max(m, y);
      }
      if ((tid & 31) == 31) scan64[tid >> 5] = (uint64_t)(int64_t)m;
      __syncthreads();
      int32_t wpre = lastp;
      for (int w = 0; w < (tid >> 5); ++w) wpre = max(wpre, (int32_t)(int64_t)scan64[w]);
      const int32_t me_ex = __shfl_up_sync(0xFFFFFFFFu, m, 1);
      const int32_t prev = max(wpre, (tid & 31) ? me_ex : -1);
      if (k < nch) {
        a.ch_bpre[ci] = run + ex;
        a.ch_bprev[ci] = prev;
      }
      int32_t tl = lastp;
      for (int w = 0; w < NT / 32; ++w) tl = max(tl, (int32_t)(int64_t)scan64[w]);
      __syncthreads();
      run += tot;
      lastp = tl;
    }
    if (tid == 0) { s_bn[b] = run; s_last[b] = lastp; }
    __syncthreads();
  }
  // q* per block
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
        if (ds > a.delta) break;  // first violation stops the descent (quant.py:110-115)
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
  {
    uint4* o4 = reinterpret_cast<uint4*>(out);
    const uint64_t n16 = P / 16;
    for (uint64_t k = tid; k < n16; k += NT) o4[k] = make_uint4(0, 0, 0, 0);
    for (uint64_t k = n16 * 16 + tid; k < P; k += NT) out[k] = 0;
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
// K7: codes, row_ptr transitions and MSB-first word assembly (chunk kernel).
struct K7Sh {
  uint32_t cur_if;
  int B;
  double vmin[MAXB], o64[MAXB], inv[MAXB];
  uint32_t q[MAXB], degen[MAXB];
  uint64_t rp[MAXB], bc[MAXB], bq[MAXB];
  uint32_t bcnt[MAXB], bpre[MAXB], rs[MAXB + 1];
  int32_t bprev[MAXB];
};

__device__ __forceinline__ void pack_words(uint32_t* out32, const uint32_t* vals, uint32_t n, uint32_t w,
                                           uint64_t b0) {
  if (n == 0) return;
  const uint64_t b1 = b0 + (uint64_t)n * w;
  const uint64_t W0 = b0 >> 5, W1 = (b1 - 1) >> 5;
  for (uint64_t W = W0 + threadIdx.x; W <= W1; W += CNT) {
    const uint64_t lo = max(W << 5, b0), hi = min((W << 5) + 32, b1);
    const uint32_t j0 = (uint32_t)(lo - b0) / w, j1 = (uint32_t)(hi - 1 - b0) / w;
    uint32_t wv = 0;
    for (uint32_t j = j0; j <= j1; ++j) {
      const int64_t t = (int64_t)(b0 + (uint64_t)j * w) - (int64_t)(W << 5);
      const int sh = 32 - (int)t - (int)w;
      const uint64_t v = vals[j];
      wv |= (uint32_t)(sh >= 0 ? (v << sh) : (v >> (-sh)));
    }
    const uint32_t le = bswap32(wv);
    if (lo == (W << 5) && hi == (W << 5) + 32) out32[W] = le;
    else if (wv) atomicOr(out32 + W, le);
  }
}

__global__ void __launch_bounds__(CNT) enc_pack(EArgs a) {
  extern __shared__ __align__(16) uint8_t dsm_raw[];
  uint32_t* dsm = reinterpret_cast<uint32_t*>(dsm_raw);
  __shared__ K7Sh sh;
  uint32_t* sv = dsm;       // codes (in place of values)
  uint32_t* sx = dsm + CH;  // flat indices, then cols
  const int tid = threadIdx.x;
  if (tid == 0) sh.cur_if = 0xFFFFFFFFu;
  __syncthreads();
  for (uint32_t c = blockIdx.x; c < (uint32_t)a.nch; c += gridDim.x) {
    const uint32_t ifi = a.ch_if[c];
    const IfInfo& f = a.info[ifi];
    IfSt& st = a.st[ifi];
    if (st.err) continue;
    if (sh.cur_if != ifi) {
      __syncthreads();
      const int B = (int)st.B;
      if (tid < B) {
        const int b = tid;
        sh.vmin[b] = (double)__uint_as_float(st.bmin[b]);
        sh.o64[b] = st.o64[b];
        sh.inv[b] = st.inv64[b];
        sh.q[b] = st.q[b];
        sh.degen[b] = st.bmin[b] == st.bmax[b] ? 1u : 0u;
        sh.rp[b] = st.off_meta[b] + kBlockMetaBytes;
        sh.bc[b] = st.bit_cols[b];
        sh.bq[b] = st.bit_codes[b];
      }
      if (tid == 0) { sh.B = B; sh.cur_if = ifi; }
      __syncthreads();
    }
    const int B = sh.B;
    if (tid < B) {
      const uint64_t ci = (uint64_t)c * a.maxb + tid;
      sh.bcnt[tid] = a.ch_bcnt[ci];
      sh.bpre[tid] = a.ch_bpre[ci];
      sh.bprev[tid] = a.ch_bprev[ci];
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t acc = 0;
      for (int b = 0; b < B; ++b) { sh.rs[b] = acc; acc += sh.bcnt[b]; }
      sh.rs[B] = acc;
    }
    __syncthreads();
    const uint32_t total = sh.rs[B];
    const uint32_t off = a.ch_off[c];
    const uint32_t* gv = lv(a, f) + off;
    const uint32_t* gx = li(a, f) + off;
    const FastDiv fk = [&] { FastDiv d; d.init(f.K); return d; }();
    // load members; codes at q* (quant.py:59-62)
    for (uint32_t k = tid; k < total; k += CNT) {
      int b = 0;
      while (b + 1 < B && sh.rs[b + 1] <= k) ++b;
      const uint32_t key = __ldcg(gv + k) & 0x7FFFFFFFu;
      const uint32_t x = __ldcg(gx + k);
      sv[k] = sh.degen[b] ? 0u : quant_code(key, sh.vmin[b], sh.o64[b], sh.inv[b], (1u << sh.q[b]) - 1u);
      sx[k] = x;
    }
    __syncthreads();
    uint8_t* out = f.out;
    // row_ptr transitions: row_ptr[r] = position of the first member with row >= r
    for (int b = 0; b < B; ++b) {
      const uint32_t n = sh.bcnt[b], r0 = sh.rs[b], p0 = sh.bpre[b];
      for (uint32_t j = tid; j < n; j += CNT) {
        const uint32_t rj = fk.div(sx[r0 + j]);
        const int32_t rprev = j ? (int32_t)fk.div(sx[r0 + j - 1]) : sh.bprev[b];
        for (int32_t r = rprev + 1; r <= (int32_t)rj; ++r) st_u32_le(out, sh.rp[b] + 4ull * (uint32_t)r, p0 + j);
      }
    }
    __syncthreads();
    for (uint32_t k = tid; k < total; k += CNT) sx[k] = fk.mod(sx[k]);
    __syncthreads();
    uint32_t* out32 = reinterpret_cast<uint32_t*>(out);
    for (int b = 0; b < B; ++b) {
      const uint32_t n = sh.bcnt[b], r0 = sh.rs[b], p0 = sh.bpre[b];
      pack_words(out32, sx + r0, n, f.cb, sh.bc[b] + (uint64_t)p0 * f.cb);
      pack_words(out32, sv + r0, n, sh.q[b], sh.bq[b] + (uint64_t)p0 * sh.q[b]);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------
// K8: CRC-32 (codec.py:316), lengths and status.
__global__ void __launch_bounds__(256) enc_crc(EArgs a) {
  constexpr int NT = 256;
  __shared__ uint32_t t4[1024];
  __shared__ uint32_t stage[16 * NT];
  __shared__ uint32_t red[NT / 32 + 2];
  const int ifi = blockIdx.x, tid = threadIdx.x;
  const IfInfo& f = a.info[ifi];
  IfSt& st = a.st[ifi];
  if (st.err) {
    if (tid == 0) {
      if (st.err == E_NONFINITE) { a.status[ifi] = SIF_ERR_NONFINITE; a.out_len[ifi] = 0; }
      else { a.status[ifi] = SIF_ERR_CAPACITY; a.out_len[ifi] = st.P; }
    }
    return;
  }
  for (int k = tid; k < 1024; k += NT) t4[k] = (&kCrcTab4[0][0])[k];
  __syncthreads();
  const uint64_t P = st.P;
  const uint32_t raw = crc_cta_staged<NT>(f.out, 4, P - 4, t4, red, stage);
  if (tid == 0) {
    st_u32_le_bytes(f.out, P - 4, crc_finish(raw, P - 8));
    a.out_len[ifi] = P;
    a.status[ifi] = SIF_OK;
  }
}

}  // namespace sif
