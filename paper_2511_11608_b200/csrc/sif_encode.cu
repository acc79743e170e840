// sif_encode.cu -- fused B200 (sm_100a) encoder for the SLICER IF codec.
//
// One thread-block cluster ("group", G CTAs, G = 1..8) encodes one IF end to end:
//
//   stream x once from HBM (128-bit loads)            atkf.py:49-55 (finite check, |x|)
//     -> bracketed candidate compaction in SMEM        (sample -> [lo,hi) bracket on |x|)
//   radix select of tau (3 x 11-bit SMEM histograms)  atkf.py:71  np.partition
//   lambda>0: strict class + second select             atkf.py:72-84
//   tie break: 64-bit radix select on splitmix keys    atkf.py:37-41, rng.py:60-68
//   kept set (stable, flat order)                      atkf.py:86-88
//   MS cut elements by rank (value desc, idx asc)      msplit.py:54-80 (no sort)
//   per-block members in CSR order (flat order)        msplit.py:83-101
//   ABQ descent with warp-reduced DS sums (float64)    quant.py:44-64, :88-115
//   .sif layout, header/meta, row_ptr, MSB-first       codec.py:283-317
//     bit packing with warp shuffles, CRC-32 combine   zlib.crc32 (codec.py:316)
//
// The result is byte-identical to serialize(encode(x, cfg, seed)) of the reference.
// Lists (candidates / kept elements / block members) live in shared memory up to
// `cap` entries per CTA and spill to a per-CTA global region beyond that.

#include <math.h>
#include <stdint.h>

#include "sif_common.cuh"

namespace sif {

constexpr int NT = 512;
constexpr int NW = NT / 32;
constexpr int MAXT = 4;        // select targets handled per batch
constexpr int HB = 2048;       // histogram bins (11-bit digits)
constexpr uint32_t kInfKey = 0xFFFFFFFFu;

struct EncArgs {
  const sif_enc_desc* descs;
  int n;
  int atkf_only;
  double s, lam, delta;
  int m_plus, m_minus, q_bit, mode;
  const uint8_t* fixed_q;  // device, m_plus + m_minus entries
  uint8_t* spill;          // per-CTA spill regions
  uint64_t spill_stride;   // bytes per CTA
  int cap;                 // list entries per CTA held in SMEM
  int maxb;                // max blocks (m_plus + m_minus)
  uint64_t* out_len;
  int32_t* status;
  int64_t* kept_out;       // atkf mode
  const uint64_t* kept_off;
  double* tau3;
};

// ---------------------------------------------------------------------------------------
// Two-tier list of (float bits, flat index) pairs.
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
// Member permutation (indices into the kept list), two-tier.
struct Perm {
  uint32_t* s;
  uint32_t* g;
  uint32_t cap;
  __device__ __forceinline__ uint32_t get(uint32_t i) const { return i < cap ? s[i] : __ldcg(g + (i - cap)); }
  __device__ __forceinline__ void set(uint32_t i, uint32_t v) const {
    if (i < cap) s[i] = v; else __stcg(g + (i - cap), v);
  }
};

// ---------------------------------------------------------------------------------------
// Group (cluster) helper: all-reduce of small u64 vectors and histogram sums via DSMEM.
struct Grp {
  uint32_t rank, size;
  uint64_t* slots;   // [2][64] u64 in smem
  int parity;
  int hpar;          // histogram double-buffer parity (cluster mode)
  __device__ __forceinline__ void sync() {
    if (size > 1) cg::this_cluster().sync();
    else __syncthreads();
  }
  __device__ __forceinline__ uint64_t* slot() { return slots + parity * 64; }
  // Sum `V` (<= 64) values the caller wrote to slot()[0..V) over the group into out[0..V)
  // (smem); optionally the exclusive prefix over lower ranks into pre[0..V).
  __device__ void allsum(int V, uint64_t* out, uint64_t* pre) {
    uint64_t* my = slot();
    sync();
    if (size == 1) {
      for (int v = threadIdx.x; v < V; v += blockDim.x) {
        out[v] = my[v];
        if (pre) pre[v] = 0;
      }
    } else {
      cg::cluster_group cl = cg::this_cluster();
      for (int v = threadIdx.x; v < V; v += blockDim.x) {
        uint64_t s = 0, p = 0;
        for (uint32_t r = 0; r < size; ++r) {
          uint64_t x = *cl.map_shared_rank(my + v, r);
          if (r < rank) p += x;
          s += x;
        }
        out[v] = s;
        if (pre) pre[v] = p;
      }
    }
    parity ^= 1;
    __syncthreads();
  }
};

// ---------------------------------------------------------------------------------------
struct Sel {
  uint64_t prefix, mask;
  uint64_t r;      // remaining rank (1-based, from the top)
  uint64_t n_gt;   // elements strictly above the final key
  uint64_t n_eq;   // elements equal to the final key
  uint32_t ok;
};

struct Shared {
  uint64_t scan[40];
  uint64_t vec[64];
  uint64_t pre[64];
  uint32_t fd_digit[MAXT];
  uint64_t fd_above[MAXT], fd_eq[MAXT];
  uint32_t fd_found[MAXT];
  // per-IF decisions
  uint32_t lo, hi, lo_neg, tau_key;
  uint32_t key_star, cls_star, tie_all, tie_skip;
  uint64_t hkey;
  uint64_t n_cand, n_kept;
  uint64_t m_eff[2], base[2], nnz[2];
  uint32_t cidx_found[MAXT];
  uint64_t run[MAXT];
  uint64_t total_len;
  uint32_t done;
};

// Find the digit d of a (group-summed) histogram such that above(d) < r <= above(d)+h[d],
// scanning from the top.  Histograms of the whole group are summed through DSMEM.
__device__ void find_digit(Grp& g, Shared& sh, const uint32_t* H, int nb, int t, uint64_t r) {
  const int per = (nb + NT - 1) / NT;  // 4 / 2 / 1
  uint64_t hv[4];
  uint64_t s = 0;
  cg::cluster_group cl = cg::this_cluster();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    hv[k] = 0;
    if (k < per) {
      int b = nb - 1 - (threadIdx.x * per + k);
      if (b >= 0) {
        if (g.size == 1) hv[k] = H[b];
        else
          for (uint32_t rr = 0; rr < g.size; ++rr) hv[k] += *cl.map_shared_rank(H + b, rr);
      }
      s += hv[k];
    }
  }
  uint64_t tot;
  uint64_t ex = block_excl_scan_u64(s, sh.scan, &tot);
  if (threadIdx.x == 0) sh.fd_found[t] = 0;
  __syncthreads();
  uint64_t cum = ex;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k < per) {
      int b = nb - 1 - (threadIdx.x * per + k);
      if (b >= 0 && cum < r && r <= cum + hv[k]) {
        sh.fd_digit[t] = (uint32_t)b;
        sh.fd_above[t] = cum;
        sh.fd_eq[t] = hv[k];
        sh.fd_found[t] = 1;
      }
      cum += hv[k];
    }
  }
  __syncthreads();
}

// Generic batched radix select ("r-th largest key") over a list of n elements.
// KeyFn(t, bits, idx, &key) -> bool : element participates in target t with key.
template <typename KeyT, class KeyFn>
__device__ void select_batch(Grp& g, Shared& sh, uint32_t* hist, const List& L, uint32_t n, int nt,
                             Sel* st, KeyFn fn) {
  constexpr int NL = sizeof(KeyT) == 8 ? 6 : 3;
  const int shifts32[3] = {21, 10, 0};
  const int widths32[3] = {11, 11, 10};
  const int shifts64[6] = {53, 42, 31, 20, 9, 0};
  const int widths64[6] = {11, 11, 11, 11, 11, 9};
  for (int lev = 0; lev < NL; ++lev) {
    const int shf = sizeof(KeyT) == 8 ? shifts64[lev] : shifts32[lev];
    const int wid = sizeof(KeyT) == 8 ? widths64[lev] : widths32[lev];
    const int nb = 1 << wid;
    uint32_t* H = hist + (g.size > 1 ? g.hpar * MAXT * HB : 0);
    g.hpar ^= 1;
    for (int i = threadIdx.x; i < nt * HB; i += NT) H[i] = 0;
    __syncthreads();
    uint64_t pf[MAXT], mk[MAXT];
#pragma unroll
    for (int t = 0; t < MAXT; ++t) {
      pf[t] = t < nt ? st[t].prefix : 0;
      mk[t] = t < nt ? st[t].mask : 0;
    }
    for (uint32_t i = threadIdx.x; i < n; i += NT) {
      uint32_t b = L.bits(i), x = L.idx(i);
#pragma unroll
      for (int t = 0; t < MAXT; ++t) {
        if (t < nt) {
          KeyT k;
          if (fn(t, b, x, k) && (((uint64_t)k & mk[t]) == pf[t]))
            atomicAdd(&H[t * HB + (int)(((uint64_t)k >> shf) & (uint64_t)(nb - 1))], 1u);
        }
      }
    }
    g.sync();
    for (int t = 0; t < nt; ++t) {
      find_digit(g, sh, H + t * HB, nb, t, st[t].r);
      if (sh.fd_found[t]) {
        st[t].prefix |= (uint64_t)sh.fd_digit[t] << shf;
        st[t].r -= sh.fd_above[t];
        st[t].n_gt += sh.fd_above[t];
        st[t].n_eq = sh.fd_eq[t];
      } else {
        st[t].ok = 0;
      }
      st[t].mask |= (uint64_t)(nb - 1) << shf;
    }
    if (g.size == 1) __syncthreads();
  }
}

__device__ __forceinline__ Sel sel_init(uint64_t r) {
  Sel s;
  s.prefix = 0; s.mask = 0; s.r = r; s.n_gt = 0; s.n_eq = 0; s.ok = 1;
  return s;
}

// quant.py:59-62 in float64: floor((v - vmin)/o64 + 0.5) clipped to [0, levels].
__device__ __forceinline__ uint32_t quant_code(uint32_t key, double vmin64, double o64, uint32_t levels) {
  double v = (double)__uint_as_float(key);
  double sc = __ddiv_rn(__dsub_rn(v, vmin64), o64);
  double f = floor(__dadd_rn(sc, 0.5));
  if (!(f > 0.0)) return 0u;
  return f >= (double)levels ? levels : (uint32_t)f;
}

// Load element e of an IF as fp32 bits.
template <int DT>
__device__ __forceinline__ uint32_t load_bits(const void* x, uint64_t e) {
  if (DT == SIF_DTYPE_F32) return __ldg(reinterpret_cast<const uint32_t*>(x) + e);
  return (uint32_t)__ldg(reinterpret_cast<const unsigned short*>(x) + e) << 16;
}

// ---------------------------------------------------------------------------------------
// Streaming pass over the CTA's slice [s0, s1): counters + stable candidate compaction.
struct Counts {
  uint64_t nz, ge_lo, ge_hi, nonfinite, maxkey;
};

template <int DT>
__device__ void stream_pass(const void* x, uint64_t T, uint64_t s0, uint64_t s1, uint32_t lo_p, uint32_t lo_n,
                            uint32_t lo_cnt, uint32_t hi_cnt, const List& L, Shared& sh, Counts& c) {
  constexpr int VEC = DT == SIF_DTYPE_F32 ? 4 : 8;
  constexpr int U = 4;
  const uint64_t CH = (uint64_t)NT * VEC * U;
  const uint64_t a0 = s0 - (s0 % VEC);
  uint64_t ncand = 0;
  for (uint64_t base = a0; base < s1; base += CH) {
    uint32_t mask[U];
    uint32_t bv[U][VEC];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t e0 = base + ((uint64_t)u * NT + threadIdx.x) * VEC;
      if (e0 + VEC <= T && e0 >= s0 && e0 + VEC <= s1) {
        uint4 v = __ldcs(reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(x) + e0 * (DT == SIF_DTYPE_F32 ? 4 : 2)));
        if (DT == SIF_DTYPE_F32) {
          bv[u][0] = v.x; bv[u][1] = v.y; bv[u][2] = v.z; bv[u][3] = v.w;
        } else {
          uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            bv[u][(2 * k) % VEC] = w[k] << 16;
            bv[u][(2 * k + 1) % VEC] = w[k] & 0xFFFF0000u;
          }
        }
        mask[u] = (1u << VEC) - 1u;
      } else {
        mask[u] = 0;
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          uint64_t e = e0 + j;
          bv[u][j] = 0;
          if (e >= s0 && e < s1 && e < T) {
            bv[u][j] = load_bits<DT>(x, e);
            mask[u] |= 1u << j;
          }
        }
      }
    }
    uint64_t packed = 0;
    uint32_t cm[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      cm[u] = 0;
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        if (mask[u] & (1u << j)) {
          uint32_t b = bv[u][j], key = b & 0x7FFFFFFFu;
          c.nz += key != 0u;
          c.ge_lo += key >= lo_cnt;
          c.ge_hi += key >= hi_cnt;
          c.nonfinite |= key >= kNonFiniteKey;
          c.maxkey = key > c.maxkey ? key : c.maxkey;
          if (key >= ((b >> 31) ? lo_n : lo_p)) cm[u] |= 1u << j;
        }
      }
      packed |= (uint64_t)__popc(cm[u]) << (16 * u);
    }
    uint64_t tot;
    uint64_t ex = block_excl_scan_u64(packed, sh.scan, &tot);
    uint64_t run = ncand;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t off = run + ((ex >> (16 * u)) & 0xFFFFull);
      const uint64_t e0 = base + ((uint64_t)u * NT + threadIdx.x) * VEC;
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        if (cm[u] & (1u << j)) {
          L.set((uint32_t)off, bv[u][j], (uint32_t)(e0 + j));
          ++off;
        }
      }
      run += (tot >> (16 * u)) & 0xFFFFull;
    }
    ncand = run;
  }
  if (threadIdx.x == 0) sh.n_cand = ncand;
  __syncthreads();
}

// Block-reduce the per-thread counters into the group slot (5 values).
__device__ void reduce_counts(Grp& g, Shared& sh, Counts& c) {
  uint64_t v[5] = {c.nz, c.ge_lo, c.ge_hi, c.nonfinite, c.maxkey};
  uint64_t* slot = g.slot();
  if (threadIdx.x < 5) slot[threadIdx.x] = 0;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    uint64_t x = v[k];
    if (k == 4) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) { uint64_t y = __shfl_xor_sync(0xFFFFFFFFu, x, o); x = y > x ? y : x; }
      if ((threadIdx.x & 31) == 0) atomicMax((unsigned long long*)&slot[k], (unsigned long long)x);
    } else if (k == 3) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x |= __shfl_xor_sync(0xFFFFFFFFu, x, o);
      if ((threadIdx.x & 31) == 0 && x) atomicOr((unsigned long long*)&slot[k], 1ull);
    } else {
      x = warp_sum_u64(x);
      if ((threadIdx.x & 31) == 0) atomicAdd((unsigned long long*)&slot[k], (unsigned long long)x);
    }
  }
  // maxkey must be max-reduced over the group, not summed: the cluster path combines it
  // through the prefix-free max below.
  g.allsum(4, sh.vec, nullptr);
  // group max of maxkey (slot of the previous parity still holds the local value)
  uint64_t mk = 0;
  {
    uint64_t* prev = g.slots + (g.parity ^ 1) * 64;
    if (g.size == 1) mk = prev[4];
    else {
      cg::cluster_group cl = cg::this_cluster();
      for (uint32_t r = 0; r < g.size; ++r) {
        uint64_t y = *cl.map_shared_rank(prev + 4, r);
        mk = y > mk ? y : mk;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) sh.vec[4] = mk;
  __syncthreads();
}

// ---------------------------------------------------------------------------------------
template <int DT>
__device__ void encode_one(const EncArgs& a, const sif_enc_desc& d, int ifi, Grp& g, uint8_t* dsm, Shared& sh) {
  const uint32_t N = d.rows, K = d.cols;
  const uint64_t T = (uint64_t)N * K;
  const uint64_t s0 = T * g.rank / g.size, s1 = T * (g.rank + 1) / g.size;
  const uint64_t kk = keep_count(a.s, T);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t cb = col_bits(K);
  const int maxb = a.maxb;

  // ---- shared memory carve-up
  uint32_t* crctab = reinterpret_cast<uint32_t*>(dsm);
  uint32_t* hist = crctab + 256;
  const int nhist = (g.size > 1 ? 2 : 1) * MAXT * HB;
  uint8_t* p = reinterpret_cast<uint8_t*>(hist + nhist);
  uint64_t* b_sum = reinterpret_cast<uint64_t*>(p); p += 8ull * maxb;
  uint64_t* b_pre = reinterpret_cast<uint64_t*>(p); p += 8ull * maxb;
  uint64_t* b_N = reinterpret_cast<uint64_t*>(p); p += 8ull * maxb;
  uint64_t* b_off = reinterpret_cast<uint64_t*>(p); p += 8ull * 4 * maxb;  // meta, rp, cols, codes
  double* b_o64 = reinterpret_cast<double*>(p); p += 8ull * maxb;
  double* b_or = reinterpret_cast<double*>(p); p += 8ull * maxb;
  uint32_t* b_n = reinterpret_cast<uint32_t*>(p); p += 4ull * maxb;
  uint32_t* b_rs = reinterpret_cast<uint32_t*>(p); p += 4ull * maxb;
  uint32_t* b_min = reinterpret_cast<uint32_t*>(p); p += 4ull * maxb;
  uint32_t* b_max = reinterpret_cast<uint32_t*>(p); p += 4ull * maxb;
  uint32_t* b_q = reinterpret_cast<uint32_t*>(p); p += 4ull * maxb;
  uint32_t* b_act = reinterpret_cast<uint32_t*>(p); p += 4ull * maxb;
  uint32_t* cut_key = reinterpret_cast<uint32_t*>(p); p += 4ull * maxb;
  uint32_t* cut_idx = reinterpret_cast<uint32_t*>(p); p += 4ull * maxb;
  uint32_t* wcnt = reinterpret_cast<uint32_t*>(p); p += 4ull * NW * maxb;
  uint32_t* woff = reinterpret_cast<uint32_t*>(p); p += 4ull * NW * maxb;
  p = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
  const uint32_t cap = (uint32_t)a.cap;
  uint8_t* spill = a.spill + a.spill_stride * ((uint64_t)ifi * g.size + g.rank);
  const uint64_t slice = s1 - s0;
  const uint64_t spill_n = slice > cap ? slice - cap : 0;
  List L;
  L.sb = reinterpret_cast<uint32_t*>(p);
  L.si = L.sb + cap;
  L.gb = reinterpret_cast<uint32_t*>(spill);
  L.gi = L.gb + spill_n;
  L.cap = cap;
  Perm M;
  M.s = L.si + cap;
  M.g = L.gi + spill_n;
  M.cap = cap;

  for (int i = tid; i < 256; i += NT) crctab[i] = kCrcTab[i];

  // ---- Phase S: sampled bracket [lo, hi) for tau (identical in every CTA of the group)
  const bool zero_mode_possible = a.atkf_only != 0;
  uint32_t lo = 1, hi = kInfKey, lo_neg = 1;
  if (T > 16384 && kk > 0 && 2 * kk <= T) {
    for (int i = tid; i < HB; i += NT) hist[i] = 0;
    __syncthreads();
    constexpr int S = 2048;
    for (int j = tid; j < S; j += NT) {
      uint64_t pos = (uint64_t)j * T / S + (T / (2 * S));
      uint32_t key = load_bits<DT>(d.x, pos) & 0x7FFFFFFFu;
      if (key && key < kNonFiniteKey) atomicAdd(&hist[key >> 20], 1u);
    }
    __syncthreads();
    const double q = (double)kk / (double)T;
    const double sd = sqrt(q * (1.0 - q) * S);
    const double rlo = ceil(q * S + 4.0 * sd + 4.0);
    const double rhi = floor(q * S - 4.0 * sd - 4.0);
    Grp g1 = g;
    g1.size = 1;  // local histogram only
    find_digit(g1, sh, hist, HB, 0, (uint64_t)rlo);
    uint32_t lo_b = sh.fd_found[0] ? sh.fd_digit[0] : 0u;
    bool lo_ok = sh.fd_found[0] != 0;
    uint32_t hi_b = 0;
    bool hi_ok = false;
    if (rhi >= 1.0) {
      find_digit(g1, sh, hist, HB, 1, (uint64_t)rhi);
      hi_ok = sh.fd_found[1] != 0;
      hi_b = sh.fd_digit[1];
    }
    lo = lo_ok ? (lo_b << 20) : 1u;
    if (lo == 0) lo = 1;
    hi = hi_ok ? ((hi_b + 1u) << 20) : kInfKey;
    if (hi_ok && hi_b + 1u >= 2048u) hi = kInfKey;
  }
  if (a.lam > 0.0 && lo > 1) {
    double t = __dmul_rn(__dsub_rn(1.0, a.lam), (double)__uint_as_float(lo));
    uint32_t k2 = __float_as_uint(__double2float_rd(t));
    lo_neg = k2 > 1 ? k2 : 1u;
  } else {
    lo_neg = lo;
  }

  // ---- Phase A: stream the slice, count, compact candidates
  Counts c;
  c.nz = c.ge_lo = c.ge_hi = c.nonfinite = c.maxkey = 0;
  stream_pass<DT>(d.x, T, s0, s1, lo, lo_neg, lo, hi, L, sh, c);
  reduce_counts(g, sh, c);
  uint64_t cnt_nz = sh.vec[0], cnt_lo = sh.vec[1], cnt_hi = sh.vec[2];
  const bool nonfinite = sh.vec[3] != 0;
  const uint32_t maxkey = (uint32_t)sh.vec[4];
  if (nonfinite) {
    if (g.rank == 0 && tid == 0) { a.status[ifi] = SIF_ERR_NONFINITE; if (!a.atkf_only) a.out_len[ifi] = 0; }
    return;
  }
  bool zero_mode = false;
  if (kk > 0) {
    uint32_t need_lo = lo;
    if (cnt_nz < kk) need_lo = zero_mode_possible ? 0u : 1u;
    else if (cnt_lo < kk) need_lo = 1u;
    if (need_lo < lo) {
      // bracket missed (or tau == 0): re-stream with everything nonzero (or every element)
      uint32_t new_hi = cnt_lo < kk ? lo : hi;
      lo = need_lo;
      lo_neg = need_lo;
      hi = new_hi;
      c.nz = c.ge_lo = c.ge_hi = c.nonfinite = c.maxkey = 0;
      stream_pass<DT>(d.x, T, s0, s1, lo, lo_neg, lo, hi, L, sh, c);
      reduce_counts(g, sh, c);
      cnt_nz = sh.vec[0]; cnt_lo = sh.vec[1]; cnt_hi = sh.vec[2];
      zero_mode = (lo == 0);
    }
  }
  const uint32_t ncand = (uint32_t)sh.n_cand;

  // ---- tau select
  uint32_t tau_key = 0;
  uint64_t n_gt = 0, n_eq = 0;
  if (kk > 0) {
    if (cnt_nz < kk) {
      tau_key = 0;
      n_gt = cnt_nz;
      n_eq = T - cnt_nz;
    } else {
      uint32_t ra, rb;
      uint64_t r, base_gt;
      if (cnt_hi >= kk || hi == kInfKey) { ra = (hi == kInfKey ? lo : hi); rb = kInfKey; r = kk; base_gt = 0; }
      else { ra = lo; rb = hi; r = kk - cnt_hi; base_gt = cnt_hi; }
      if (ra == 0) ra = 1;
      Sel st = sel_init(r);
      select_batch<uint32_t>(g, sh, hist, L, ncand, 1, &st,
                             [&](int, uint32_t b, uint32_t, uint32_t& k) {
                               k = b & 0x7FFFFFFFu;
                               return k >= ra && k < rb;
                             });
      tau_key = (uint32_t)st.prefix;
      n_gt = base_gt + st.n_gt;
      n_eq = st.n_eq;
    }
  }
  const double tau = kk > 0 ? (double)__uint_as_float(tau_key) : (double)__uint_as_float(maxkey);
  const double tau_p = __dmul_rn(__dadd_rn(1.0, a.lam), tau);
  const double tau_m = -__dmul_rn(__dsub_rn(1.0, a.lam), tau);

  // ---- lambda > 0: strict class (atkf.py:75-84)
  const bool use_cls = a.lam > 0.0 && kk > 0 && (tau_key > 0 || zero_mode);
  uint32_t key_star = tau_key, cls_star = 0;
  uint64_t r_t = kk - n_gt;  // ties to take at key_star
  auto strict_of = [&](uint32_t b) -> uint32_t {
    double v = (double)__uint_as_float(b);
    return (v > tau_p || v < tau_m) ? 1u : 0u;
  };
  if (use_cls) {
    uint64_t ns = 0;
    for (uint32_t i = tid; i < ncand; i += NT) ns += strict_of(L.bits(i));
    ns = warp_sum_u64(ns);
    uint64_t* slot = g.slot();
    if (tid == 0) slot[0] = 0;
    __syncthreads();
    if (lane == 0) atomicAdd((unsigned long long*)&slot[0], (unsigned long long)ns);
    g.allsum(1, sh.vec, nullptr);
    const uint64_t n_strict = sh.vec[0];
    uint64_t r;
    if (n_strict >= kk) { cls_star = 1; r = kk; }
    else { cls_star = 0; r = kk - n_strict; }
    const uint32_t cs = cls_star;
    Sel st = sel_init(r);
    select_batch<uint32_t>(g, sh, hist, L, ncand, 1, &st,
                           [&](int, uint32_t b, uint32_t, uint32_t& k) {
                             k = b & 0x7FFFFFFFu;
                             return strict_of(b) == cs;
                           });
    key_star = (uint32_t)st.prefix;
    n_eq = st.n_eq;
    r_t = st.r;  // remaining rank inside the tie set
  }
  // ---- tie break by splitmix64 key (rng.py:60-68), smallest keys first
  // tie modes: all ties kept / none / zero ties (never reach the payload) / by hash
  bool tie_all = r_t >= n_eq;
  bool tie_none = !tie_all && r_t == 0;
  bool tie_skip = (!zero_mode && key_star == 0);
  uint64_t hkey = 0;
  if (kk > 0 && !tie_all && !tie_none && !tie_skip) {
    const uint32_t ks = key_star, cs = cls_star;
    const bool uc = use_cls;
    const uint64_t seed = d.seed;
    Sel st = sel_init(r_t);
    select_batch<uint64_t>(g, sh, hist, L, ncand, 1, &st,
                           [&](int, uint32_t b, uint32_t x, uint64_t& k) {
                             if ((b & 0x7FFFFFFFu) != ks) return false;
                             if (uc && strict_of(b) != cs) return false;
                             k = ~splitmix(seed, x);
                             return true;
                           });
    hkey = st.prefix;
  }

  // ---- kept set: stable in-place compaction of the candidate list (atkf.py:83-88)
  uint32_t nkept = 0;
  uint64_t cnt_sign[2] = {0, 0};
  {
    const uint32_t ks = key_star, cs = cls_star;
    const bool uc = use_cls, ta = tie_all, tsk = tie_skip || tie_none;
    const uint64_t hk = hkey, seed = d.seed;
    auto kept_of = [&](uint32_t b, uint32_t x) -> bool {
      if (kk == 0) return false;
      uint32_t key = b & 0x7FFFFFFFu;
      if (!zero_mode && key == 0) return false;
      if (uc) {
        uint32_t cl = strict_of(b);
        if (cl != cs) return cl > cs;
      }
      if (key != ks) return key > ks;
      if (tsk) return false;
      if (ta) return true;
      return ~splitmix(seed, x) >= hk;
    };
    uint32_t run = 0;
    uint64_t sp = 0, sm = 0;
    for (uint32_t base = 0; base < ncand; base += NT) {
      uint32_t i = base + tid;
      uint32_t b = 0, x = 0;
      bool k = false;
      if (i < ncand) {
        b = L.bits(i);
        x = L.idx(i);
        k = kept_of(b, x);
      }
      uint64_t tot;
      uint64_t ex = block_excl_scan_u64(k ? 1ull : 0ull, sh.scan, &tot);
      if (k) {
        L.set(run + (uint32_t)ex, b, x);
        if ((b & 0x7FFFFFFFu) != 0) { if (b >> 31) ++sm; else ++sp; }
      }
      run += (uint32_t)tot;
      __syncthreads();
    }
    nkept = run;
    sp = warp_sum_u64(sp);
    sm = warp_sum_u64(sm);
    uint64_t* slot = g.slot();
    if (tid < 3) slot[tid] = 0;
    __syncthreads();
    if (lane == 0) {
      atomicAdd((unsigned long long*)&slot[0], (unsigned long long)sp);
      atomicAdd((unsigned long long*)&slot[1], (unsigned long long)sm);
    }
    if (tid == 0) slot[2] = nkept;
    g.allsum(3, sh.vec, sh.pre);
    cnt_sign[0] = sh.vec[0];
    cnt_sign[1] = sh.vec[1];
  }
  const uint64_t kept_pre = sh.pre[2];

  if (a.atkf_only) {
    int64_t* out = a.kept_out + a.kept_off[ifi] + kept_pre;
    for (uint32_t i = tid; i < nkept; i += NT) out[i] = (int64_t)L.idx(i);
    if (g.rank == 0 && tid == 0) {
      a.tau3[3 * ifi + 0] = tau;
      a.tau3[3 * ifi + 1] = tau_p;
      a.tau3[3 * ifi + 2] = tau_m;
      a.status[ifi] = SIF_OK;
    }
    return;
  }

  // ---- MS: plane sizes and cut elements (msplit.py:54-80)
  const int mcfg[2] = {a.m_plus, a.m_minus};
  uint64_t meff[2], base[2];
  for (int s = 0; s < 2; ++s) {
    uint64_t nz = cnt_sign[s];
    uint64_t m = (uint64_t)mcfg[s];
    meff[s] = nz < m ? nz : m;
    if (meff[s] < 1) meff[s] = 1;
    base[s] = nz / meff[s];
  }
  const int B = (int)(meff[0] + meff[1]);
  // cuts: sign s, j = 1..meff[s]-1 at 0-based rank j*base[s]; stored at cut index
  // (s ? meff[0]-1 : 0) + j - 1
  const int ncut = B - 2;
  for (int c0 = 0; c0 < ncut; c0 += MAXT) {
    const int nt = ncut - c0 < MAXT ? ncut - c0 : MAXT;
    Sel st[MAXT];
    uint32_t sg[MAXT];
    uint64_t rank0[MAXT];
    for (int t = 0; t < MAXT; ++t) {
      int ci = c0 + t;
      if (t < nt) {
        int s = ci < (int)meff[0] - 1 ? 0 : 1;
        int j = (s == 0 ? ci : ci - ((int)meff[0] - 1)) + 1;
        sg[t] = s;
        rank0[t] = (uint64_t)j * base[s];
        st[t] = sel_init(rank0[t] + 1);
      } else {
        sg[t] = 0; rank0[t] = 0; st[t] = sel_init(1);
      }
    }
    select_batch<uint32_t>(g, sh, hist, L, nkept, nt, st,
                           [&](int t, uint32_t b, uint32_t, uint32_t& k) {
                             k = b & 0x7FFFFFFFu;
                             return (b >> 31) == sg[t] && k != 0;
                           });
    // idx resolution: the (rank0 - n_gt)-th (0-based) element, in flat order, among the
    // kept elements of the cut's sign whose key equals the cut key (msplit.py:64 ties).
    uint32_t ck[MAXT];
    for (int t = 0; t < MAXT; ++t) ck[t] = (uint32_t)st[t].prefix;
    uint64_t* slot = g.slot();
    if (tid < MAXT) slot[tid] = 0;
    __syncthreads();
    {
      uint32_t cnt[MAXT] = {0, 0, 0, 0};
      for (uint32_t i = tid; i < nkept; i += NT) {
        uint32_t b = L.bits(i);
#pragma unroll
        for (int t = 0; t < MAXT; ++t)
          if (t < nt && (b >> 31) == sg[t] && (b & 0x7FFFFFFFu) == ck[t]) ++cnt[t];
      }
#pragma unroll
      for (int t = 0; t < MAXT; ++t) {
        uint32_t v = __reduce_add_sync(0xFFFFFFFFu, cnt[t]);
        if (lane == 0 && v) atomicAdd((unsigned long long*)&slot[t], (unsigned long long)v);
      }
    }
    g.allsum(MAXT, sh.vec, sh.pre);
    uint64_t want[MAXT];
    bool mine[MAXT];
    {
      const uint64_t* prev = g.slots + (g.parity ^ 1) * 64;  // this CTA's local counts
      for (int t = 0; t < MAXT; ++t) {
        const uint64_t w = rank0[t] - st[t].n_gt;
        mine[t] = t < nt && w >= sh.pre[t] && w < sh.pre[t] + prev[t];
        want[t] = w - sh.pre[t];
      }
    }
    if (tid < MAXT) { sh.cidx_found[tid] = 0; sh.run[tid] = 0; }
    __syncthreads();
    for (uint32_t base2 = 0; base2 < nkept; base2 += NT) {
      const uint32_t i = base2 + tid;
      const uint32_t b = i < nkept ? L.bits(i) : 0u;
      uint64_t pk = 0;
      if (i < nkept)
        for (int t = 0; t < MAXT; ++t)
          if (mine[t] && (b >> 31) == sg[t] && (b & 0x7FFFFFFFu) == ck[t]) pk |= 1ull << (16 * t);
      uint64_t tot;
      const uint64_t ex = block_excl_scan_u64(pk, sh.scan, &tot);
      for (int t = 0; t < MAXT; ++t)
        if (((pk >> (16 * t)) & 1ull) && sh.run[t] + ((ex >> (16 * t)) & 0xFFFFull) == want[t]) {
          sh.cidx_found[t] = 1;
          cut_idx[c0 + t] = L.idx(i);
        }
      __syncthreads();
      if (tid < MAXT) sh.run[tid] += (tot >> (16 * tid)) & 0xFFFFull;
      __syncthreads();
    }
    uint64_t* slot2 = g.slot();
    if (tid < MAXT) slot2[tid] = (tid < nt && sh.cidx_found[tid]) ? (uint64_t)cut_idx[c0 + tid] + 1ull : 0ull;
    g.allsum(MAXT, sh.vec, nullptr);
    if (tid < nt) {
      cut_key[c0 + tid] = ck[tid];
      cut_idx[c0 + tid] = (uint32_t)(sh.vec[tid] - 1ull);
    }
    __syncthreads();
  }
  const int ncut0 = (int)meff[0] - 1;
  auto block_of = [&](uint32_t b, uint32_t x) -> int {
    uint32_t key = b & 0x7FFFFFFFu;
    int s = (int)(b >> 31);
    int c0 = s ? ncut0 : 0, cn = s ? ncut : ncut0;
    int blk = 0;
    for (int c = c0; c < cn; ++c) {
      uint32_t k2 = cut_key[c];
      if (key < k2 || (key == k2 && x >= cut_idx[c])) ++blk;
      else break;
    }
    return (s ? (int)meff[0] : 0) + blk;
  };

  // ---- members per block in flat (CSR) order: warp-segmented stable walk
  {
    const uint32_t seg = (nkept + NW - 1) / NW;
    const uint32_t w0 = wid * seg, w1 = (w0 + seg < nkept) ? w0 + seg : nkept;
    for (int b = lane; b < B; b += 32) wcnt[wid * maxb + b] = 0;
    __syncwarp();
    for (uint32_t i = w0; i < w1; i += 32) {
      uint32_t e = i + lane;
      int blk = e < w1 ? block_of(L.bits(e), L.idx(e)) : -1;
      uint32_t peers = __match_any_sync(0xFFFFFFFFu, blk);
      if (blk >= 0 && lane == __ffs(peers) - 1) wcnt[wid * maxb + blk] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    for (int b = tid; b < B; b += NT) {
      uint32_t acc = 0;
      for (int w = 0; w < NW; ++w) {
        woff[w * maxb + b] = acc;
        acc += wcnt[w * maxb + b];
      }
      b_n[b] = acc;
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t acc = 0;
      for (int b = 0; b < B; ++b) { b_rs[b] = acc; acc += b_n[b]; }
    }
    for (int b = lane; b < B; b += 32) wcnt[wid * maxb + b] = 0;
    __syncthreads();
    for (uint32_t i = w0; i < w1; i += 32) {
      uint32_t e = i + lane;
      int blk = e < w1 ? block_of(L.bits(e), L.idx(e)) : -1;
      uint32_t peers = __match_any_sync(0xFFFFFFFFu, blk);
      if (blk >= 0) {
        uint32_t rank = woff[wid * maxb + blk] + wcnt[wid * maxb + blk] + __popc(peers & ((1u << lane) - 1u));
        M.set(b_rs[blk] + rank, e);
      }
      __syncwarp();
      if (blk >= 0 && lane == __ffs(peers) - 1) wcnt[wid * maxb + blk] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    // group prefix of per-block counts + block min/max keys
    for (int b0 = 0; b0 < B; b0 += 64) {
      int nb = B - b0 < 64 ? B - b0 : 64;
      uint64_t* slot = g.slot();
      if (tid < nb) slot[tid] = b_n[b0 + tid];
      g.allsum(nb, sh.vec, sh.pre);
      if (tid < nb) { b_N[b0 + tid] = sh.vec[tid]; b_pre[b0 + tid] = sh.pre[tid]; }
      __syncthreads();
    }
  }
  // block min / max keys (v_min, v_max of quant.py:50-51)
  for (int b = tid; b < B; b += NT) { b_min[b] = 0x7FFFFFFFu; b_max[b] = 0u; }
  __syncthreads();
  for (int b = 0; b < B; ++b) {
    uint32_t mn = 0x7FFFFFFFu, mx = 0;
    for (uint32_t i = tid; i < b_n[b]; i += NT) {
      uint32_t k = L.bits(M.get(b_rs[b] + i)) & 0x7FFFFFFFu;
      mn = k < mn ? k : mn;
      mx = k > mx ? k : mx;
    }
    mn = __reduce_min_sync(0xFFFFFFFFu, mn);
    mx = __reduce_max_sync(0xFFFFFFFFu, mx);
    if (lane == 0) { atomicMin(&b_min[b], mn); atomicMax(&b_max[b], mx); }
  }
  __syncthreads();
  if (g.size > 1) {
    for (int b0 = 0; b0 < B; b0 += 32) {
      int nb = B - b0 < 32 ? B - b0 : 32;
      uint64_t* slot = g.slot();
      // pack (0x7FFFFFFF - min) and max so that a single max-reduction works via sums of
      // one-hot contributions is not possible; gather explicitly instead
      if (tid < nb) { slot[tid] = b_min[b0 + tid]; slot[32 + tid] = b_max[b0 + tid]; }
      g.sync();
      cg::cluster_group cl = cg::this_cluster();
      if (tid < nb) {
        uint32_t mn = 0x7FFFFFFFu, mx = 0;
        for (uint32_t r = 0; r < g.size; ++r) {
          uint32_t a0 = (uint32_t)*cl.map_shared_rank(slot + tid, r);
          uint32_t a1 = (uint32_t)*cl.map_shared_rank(slot + 32 + tid, r);
          mn = a0 < mn ? a0 : mn;
          mx = a1 > mx ? a1 : mx;
        }
        b_min[b0 + tid] = mn;
        b_max[b0 + tid] = mx;
      }
      g.parity ^= 1;
      __syncthreads();
    }
  }

  // ---- ABQ (quant.py:102-115) / fixed Q (codec.py:180-181, :194-200)
  for (int b = tid; b < B; b += NT) {
    const int s = b < (int)meff[0] ? 0 : 1;
    const int j = s ? b - (int)meff[0] : b;
    const bool empty = b_N[b] == 0;
    const bool degen = !empty && b_min[b] == b_max[b];
    uint32_t q;
    if (a.mode == SIF_MODE_FIXED) q = a.fixed_q[(s ? a.m_plus : 0) + j];
    else if (empty) q = (uint32_t)a.q_bit;
    else if (degen) q = 1;
    else q = 0;  // to be searched
    b_q[b] = q;
    b_act[b] = q == 0 ? 1u : 0u;
    if (q == 0) b_q[b] = (uint32_t)a.q_bit;
    const double vmin = (double)__uint_as_float(b_min[b]), vmax = (double)__uint_as_float(b_max[b]);
    b_or[b] = __ddiv_rn(__dsub_rn(vmax, vmin), (double)((1u << a.q_bit) - 1u));
  }
  __syncthreads();
  if (a.mode != SIF_MODE_FIXED) {
    for (int q = a.q_bit - 1; q >= 1; --q) {
      int any = 0;
      for (int b = 0; b < B; ++b) any |= (int)b_act[b];
      if (!any) break;
      const uint32_t lv = (1u << q) - 1u, lref = (1u << a.q_bit) - 1u;
      const int shift = a.q_bit - q;
      for (int b = tid; b < B; b += NT) {
        b_sum[b] = 0;
        const double vmin = (double)__uint_as_float(b_min[b]), vmax = (double)__uint_as_float(b_max[b]);
        b_o64[b] = __ddiv_rn(__dsub_rn(vmax, vmin), (double)lv);
      }
      __syncthreads();
      for (int b = 0; b < B; ++b) {
        if (!b_act[b]) continue;
        const double vmin = (double)__uint_as_float(b_min[b]);
        const double oq = b_o64[b], orf = b_or[b];
        uint32_t acc = 0;
        for (uint32_t i = tid; i < b_n[b]; i += NT) {
          uint32_t k = L.bits(M.get(b_rs[b] + i)) & 0x7FFFFFFFu;
          uint32_t cr = quant_code(k, vmin, orf, lref) >> shift;
          uint32_t cq = quant_code(k, vmin, oq, lv);
          acc += cr > cq ? cr - cq : cq - cr;
        }
        acc = __reduce_add_sync(0xFFFFFFFFu, acc);
        if (lane == 0 && acc) atomicAdd((unsigned long long*)&b_sum[b], (unsigned long long)acc);
      }
      __syncthreads();
      for (int b0 = 0; b0 < B; b0 += 64) {
        int nb = B - b0 < 64 ? B - b0 : 64;
        uint64_t* slot = g.slot();
        if (tid < nb) slot[tid] = b_sum[b0 + tid];
        g.allsum(nb, sh.vec, nullptr);
        if (tid < nb) {
          int b = b0 + tid;
          if (b_act[b]) {
            double ds = __ddiv_rn((double)sh.vec[tid], (double)b_N[b]);
            if (ds > a.delta) b_act[b] = 0;  // first violation stops the descent
            else { b_q[b] = (uint32_t)q; if (q == 1) b_act[b] = 0; }
          }
        }
        __syncthreads();
      }
    }
  }

  // ---- layout (codec.py:269-280)
  if (tid == 0) {
    uint64_t pos = kHeaderBytes + (a.mode == SIF_MODE_FIXED ? (uint64_t)B : 0ull);
    for (int b = 0; b < B; ++b) {
      b_off[4 * b + 0] = pos;
      b_off[4 * b + 1] = pos + kBlockMetaBytes;
      pos += kBlockMetaBytes + 4ull * ((uint64_t)N + 1ull);
      b_off[4 * b + 2] = pos;
      pos += (b_N[b] * cb + 7ull) / 8ull;
      b_off[4 * b + 3] = pos;
      pos += (b_N[b] * b_q[b] + 7ull) / 8ull;
    }
    sh.total_len = pos + kCrcBytes;
  }
  for (int b = tid; b < B; b += NT) {
    const double vmin = (double)__uint_as_float(b_min[b]), vmax = (double)__uint_as_float(b_max[b]);
    const bool degen = b_N[b] == 0 || b_min[b] == b_max[b];
    b_o64[b] = degen ? 1.0 : __ddiv_rn(__dsub_rn(vmax, vmin), (double)((1u << b_q[b]) - 1u));
  }
  __syncthreads();
  const uint64_t P = sh.total_len;
  if (P > d.out_cap) {
    if (g.rank == 0 && tid == 0) { a.status[ifi] = SIF_ERR_CAPACITY; a.out_len[ifi] = P; }
    return;
  }
  uint8_t* out = d.out;
  // ---- zero-fill this CTA's share of the payload
  {
    const uint64_t z0 = P * g.rank / g.size, z1 = P * (g.rank + 1) / g.size;
    uint64_t za = (z0 + 15) & ~15ull, zb = z1 & ~15ull;
    if (za > zb) { za = z1; zb = z1; }
    for (uint64_t i = z0 + tid; i < za && i < z1; i += NT) out[i] = 0;
    for (uint64_t i = zb + tid; i < z1; i += NT) if (i >= za) out[i] = 0;
    uint4* o4 = reinterpret_cast<uint4*>(out);
    for (uint64_t i = za / 16 + tid; i < zb / 16; i += NT) o4[i] = make_uint4(0, 0, 0, 0);
  }
  __threadfence();
  g.sync();

  // ---- header, Q vector, block meta (codec.py:285-306) by rank 0
  if (g.rank == 0) {
    if (tid == 0) {
      uint8_t h[32];
      h[0] = 'S'; h[1] = 'I'; h[2] = 'F'; h[3] = '1';
      h[4] = 1; h[5] = 0;
      uint32_t f[2] = {N, K};
      for (int k = 0; k < 4; ++k) { h[6 + k] = (uint8_t)(f[0] >> (8 * k)); h[10 + k] = (uint8_t)(f[1] >> (8 * k)); }
      uint32_t s32 = __float_as_uint(__double2float_rn(a.s));
      uint32_t l32 = __float_as_uint(__double2float_rn(a.lam));
      uint32_t d32 = __float_as_uint(__double2float_rn(a.delta));
      for (int k = 0; k < 4; ++k) {
        h[14 + k] = (uint8_t)(s32 >> (8 * k));
        h[18 + k] = (uint8_t)(l32 >> (8 * k));
        h[23 + k] = (uint8_t)(d32 >> (8 * k));
      }
      h[22] = (uint8_t)a.q_bit;
      h[27] = (uint8_t)a.mode;
      h[28] = (uint8_t)meff[0]; h[29] = (uint8_t)(meff[0] >> 8);
      h[30] = (uint8_t)meff[1]; h[31] = (uint8_t)(meff[1] >> 8);
      for (int k = 0; k < 32; ++k) out[k] = h[k];
    }
    if (a.mode == SIF_MODE_FIXED)
      for (int b = tid; b < B; b += NT) out[kHeaderBytes + b] = (uint8_t)b_q[b];
    for (int b = tid; b < B; b += NT) {
      const uint64_t o = b_off[4 * b];
      out[o] = (uint8_t)b_q[b];
      st_u32_le_bytes(out, o + 1, __float_as_uint(b_N[b] == 0 ? 1.0f : __double2float_rn(b_o64[b])));
      st_u32_le_bytes(out, o + 5, b_N[b] == 0 ? 0u : b_min[b]);
      st_u32_le_bytes(out, o + 9, (uint32_t)b_N[b]);
    }
  }
  // ---- row_ptr (msplit.py:97-100): rows whose start r*K lies in [s0, s1) (+ row N last)
  {
    const uint64_t r0 = (s0 + K - 1) / K;
    uint64_t r1 = (s1 + K - 1) / K;  // exclusive
    if (r1 > N) r1 = N;
    const bool last = g.rank == g.size - 1;
    const uint64_t nr = (r1 > r0 ? r1 - r0 : 0) + (last ? 1 : 0);
    const uint64_t tot = nr * (uint64_t)B;
    for (uint64_t w = tid; w < tot; w += NT) {
      const int b = (int)(w / nr);
      const uint64_t rr = w % nr;
      const uint64_t r = (last && rr == nr - 1) ? (uint64_t)N : r0 + rr;
      uint32_t val;
      if (r == N) {
        val = (uint32_t)b_N[b];
      } else {
        const uint64_t bound = r * K;
        uint32_t lo2 = 0, hi2 = b_n[b];
        while (lo2 < hi2) {
          uint32_t mid = (lo2 + hi2) >> 1;
          if ((uint64_t)L.idx(M.get(b_rs[b] + mid)) < bound) lo2 = mid + 1; else hi2 = mid;
        }
        val = (uint32_t)(b_pre[b] + lo2);
      }
      st_u32_le_bytes(out, b_off[4 * b + 1] + 4ull * r, val);
    }
  }
  // ---- cols / codes: MSB-first bit packing with warp shuffles (bitstream.py:12-30)
  {
    uint32_t* out32 = reinterpret_cast<uint32_t*>(out);
    for (int b = 0; b < B; ++b) {
      const uint64_t nloc = b_n[b];
      if (nloc == 0) continue;
      const uint64_t pre = b_pre[b];
      const uint64_t gfirst = pre / 32, glast = (pre + nloc - 1) / 32;
      const double vmin = (double)__uint_as_float(b_min[b]);
      const double o64 = b_o64[b];
      const uint32_t qb = b_q[b], lv = (1u << qb) - 1u;
      const bool degen = b_min[b] == b_max[b];
      for (int sec = 0; sec < 2; ++sec) {
        const uint32_t w = sec == 0 ? cb : qb;
        const uint64_t secbit = 8ull * b_off[4 * b + 2 + sec];
        const int kmax = (int)(31u / w) + 2 < 33 ? (int)(31u / w) + 2 : 33;
        for (uint64_t gi = gfirst + wid; gi <= glast; gi += NW) {
          const uint64_t p0 = gi * 32ull;
          const uint64_t pp = p0 + lane;
          const bool valid = pp >= pre && pp < pre + nloc;
          uint32_t val = 0;
          if (valid) {
            uint32_t li = M.get(b_rs[b] + (uint32_t)(pp - pre));
            if (sec == 0) val = L.idx(li) % K;
            else val = degen ? 0u : quant_code(L.bits(li) & 0x7FFFFFFFu, vmin, o64, lv);
          }
          const uint64_t f_lo = (pre > p0 ? pre : p0) - p0;
          const uint64_t f_hi = ((pre + nloc) < (p0 + 32) ? (pre + nloc) : (p0 + 32)) - p0;
          const uint64_t Gs = secbit + p0 * w;
          const uint64_t own_lo = Gs + f_lo * w, own_hi = Gs + f_hi * w;
          const uint64_t a0w = own_lo >> 5, a1w = (own_hi - 1) >> 5;
          const uint32_t nwords = (uint32_t)(a1w - a0w + 1);
          for (uint32_t wb = 0; wb < nwords; wb += 32) {
            const uint32_t j = wb + lane;
            const uint64_t W = (a0w + j) * 32ull;
            const int64_t fstart = W > Gs ? (int64_t)((W - Gs) / w) : 0;
            uint32_t acc = 0;
            for (int k = 0; k < kmax; ++k) {
              const int64_t f = fstart + k;
              const int src = f < 31 ? (int)f : 31;
              const uint32_t fv = __shfl_sync(0xFFFFFFFFu, val, src);
              if (j < nwords && f <= 31) {
                const int64_t pos = (int64_t)(Gs + (uint64_t)f * w) - (int64_t)W;
                if (pos < 32 && pos + (int64_t)w > 0) {
                  const int sh2 = 64 - (int)w - (int)pos;
                  const uint64_t v64 = sh2 >= 64 ? 0ull : ((uint64_t)fv << sh2);
                  acc |= (uint32_t)(v64 >> 32);
                }
              }
            }
            if (j < nwords) {
              const bool full = W >= own_lo && W + 32 <= own_hi;
              if (full) out32[a0w + j] = bswap32(acc);
              else if (acc) atomicOr(out32 + a0w + j, bswap32(acc));
            }
          }
        }
      }
    }
  }
  __threadfence();
  g.sync();

  // ---- CRC-32 over bytes [4, P-4) (codec.py:316), chunked + GF(2) combine
  {
    const uint64_t Lc = P - 8;
    const uint64_t c0 = 4 + Lc * g.rank / g.size, c1 = 4 + Lc * (g.rank + 1) / g.size;
    const uint64_t n_me = c1 - c0;
    const uint64_t t0 = c0 + n_me * tid / NT, t1 = c0 + n_me * (tid + 1) / NT;
    uint32_t raw = crc_raw_range(out, t0, t1, crctab);
    raw = crc_shift(raw, (P - 4) - t1);
    raw = warp_xor(raw);
    uint64_t* slot = g.slot();
    if (tid == 0) slot[0] = 0;
    __syncthreads();
    if (lane == 0) atomicXor((unsigned long long*)&slot[0], (unsigned long long)raw);
    // xor-combine across the group: use allsum on one-hot-free path (gather explicitly)
    g.sync();
    uint32_t total = 0;
    if (g.size == 1) total = (uint32_t)slot[0];
    else {
      cg::cluster_group cl = cg::this_cluster();
      for (uint32_t r = 0; r < g.size; ++r) total ^= (uint32_t)*cl.map_shared_rank(slot, r);
    }
    g.parity ^= 1;
    if (g.rank == 0 && tid == 0) {
      const uint32_t crc = crc_finish(total, Lc);
      st_u32_le_bytes(out, P - 4, crc);
      a.out_len[ifi] = P;
      a.status[ifi] = SIF_OK;
    }
  }
}

__global__ void __launch_bounds__(NT, 1) sif_encode_kernel(EncArgs a) {
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ Shared sh;
  __shared__ uint64_t slots[128];
  Grp g;
  {
    cg::cluster_group cl = cg::this_cluster();
    g.rank = cl.block_rank();
    g.size = cl.num_blocks();
  }
  g.slots = slots;
  g.parity = 0;
  g.hpar = 0;
  const int ifi = blockIdx.x / g.size;
  if (ifi >= a.n) return;
  const sif_enc_desc d = a.descs[ifi];
  if (d.dtype == SIF_DTYPE_BF16) encode_one<SIF_DTYPE_BF16>(a, d, ifi, g, dsm, sh);
  else encode_one<SIF_DTYPE_F32>(a, d, ifi, g, dsm, sh);
  if (g.size > 1) cg::this_cluster().sync();  // keep DSMEM alive until all peers are done
}

}  // namespace sif
