// sif_encode.cu -- fused B200 (sm_100a) encoder for the SLICER IF codec.
//
// One thread-block cluster ("group", G CTAs, G = 1..8) encodes one IF end to end; every
// CTA owns a contiguous flat slice of the IF.  Phases (reference semantics cited):
//
//   S  sample 4096 elements -> bracket [lo, hi) around the k-th |x|     (speculation only)
//   A  stream the slice once from HBM (128-bit loads, software-pipelined):
//      NaN/Inf check (atkf.py:49-51), counts, stable compaction of candidates |x| >= lo
//   B  exact select of tau and of the tie cut: histogram -> gather the target bin ->
//      rank by (|x| desc, splitmix64 asc) (atkf.py:37-41, :71-84, rng.py:60-68)
//   C  kept set, stable in flat order (atkf.py:83-88)
//   D  MS cut elements at ranks j*base by (value desc, flat idx asc) (msplit.py:54-80)
//   E  block members in CSR order (warp-segmented stable walk)           (msplit.py:83-101)
//   F  v_min / v_max per block, G  ABQ descent (quant.py:44-64, :88-115)
//   H  .sif layout, header/meta, row_ptr, MSB-first word packing, CRC-32 (codec.py:283-317)
//
// The output is byte-identical to serialize(encode(x, cfg, seed)) of the reference.
// Lists live in shared memory up to `cap` entries per CTA and spill to a per-CTA global
// region beyond that.

#include <math.h>
#include <stdint.h>

#include "sif_common.cuh"

namespace sif {

constexpr int HB = 2048;           // histogram bins (11-bit digits)
constexpr int GCAP = 1024;         // gather capacity (group total) for exact ranking
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
  int scratch_words;       // selection scratch (histograms + gather buffers), u32 words
  uint64_t* out_len;
  int32_t* status;
  int64_t* kept_out;       // atkf mode
  const uint64_t* kept_off;
  double* tau3;
  uint64_t* prof;          // optional per-IF phase timestamps (globaltimer ns), 32 per IF
};

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SIF_PHASE(k) \
  do { if (a.prof && g.rank == 0 && threadIdx.x == 0) a.prof[(uint64_t)ifi * 32 + (k)] = gtimer(); } while (0)

// ---------------------------------------------------------------------------------------
// Two-tier list of (float bits, flat index) pairs.
struct List {
  uint32_t* sb;
  uint32_t* si;
  uint32_t* gb;
  uint32_t* gi;
  uint32_t cap;
  __device__ __forceinline__ uint32_t bits(uint32_t i) const { return *(i < cap ? sb + i : gb + (i - cap)); }
  __device__ __forceinline__ uint32_t idx(uint32_t i) const { return *(i < cap ? si + i : gi + (i - cap)); }
  __device__ __forceinline__ void set(uint32_t i, uint32_t b, uint32_t x) const {
    if (i < cap) { sb[i] = b; si[i] = x; }
    else { __stcg(gb + (i - cap), b); __stcg(gi + (i - cap), x); }
  }
  __device__ __forceinline__ void set_bits(uint32_t i, uint32_t b) const {
    if (i < cap) sb[i] = b; else __stcg(gb + (i - cap), b);
  }
};
struct Perm {
  uint32_t* s;
  uint32_t* g;
  uint32_t cap;
  __device__ __forceinline__ uint32_t get(uint32_t i) const { return *(i < cap ? s + i : g + (i - cap)); }
  __device__ __forceinline__ void set(uint32_t i, uint32_t v) const {
    if (i < cap) s[i] = v; else __stcg(g + (i - cap), v);
  }
};

// Visit every list element (order-free).  Shared-memory-resident lists are read with
// 128-bit loads (4 elements per thread per step) and no per-element spill branch.
template <int NT, class F>
__device__ __forceinline__ void list_foreach(const List& L, uint32_t n, F f) {
  if (n <= L.cap) {
    const uint32_t n4 = n & ~3u;
    for (uint32_t i = threadIdx.x * 4; i < n4; i += NT * 4) {
      const uint4 b4 = *reinterpret_cast<const uint4*>(L.sb + i);
      const uint4 x4 = *reinterpret_cast<const uint4*>(L.si + i);
      f(b4.x, x4.x);
      f(b4.y, x4.y);
      f(b4.z, x4.z);
      f(b4.w, x4.w);
    }
    for (uint32_t i = n4 + threadIdx.x; i < n; i += NT) f(L.sb[i], L.si[i]);
  } else {
    for (uint32_t i = threadIdx.x; i < n; i += NT) f(L.bits(i), L.idx(i));
  }
}

// ---------------------------------------------------------------------------------------
// Group (cluster) helper: small-vector all-reduce and DSMEM access.
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
  // Sum V (<= 64) values the caller wrote to slot()[0..V) over the group into out[0..V);
  // optionally the exclusive prefix over lower ranks into pre[0..V).
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
          const uint64_t x = *cl.map_shared_rank(my + v, r);
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

struct GatE {
  uint32_t key;
  uint32_t idx;
  uint64_t sec;
};

struct Shared {
  uint64_t scan[40];
  uint64_t vec[64];
  uint64_t pre[64];
  uint32_t red[40];
  uint32_t fd_digit;
  uint64_t fd_above, fd_eq;
  uint32_t fd_found;
  uint32_t gcount;
  uint32_t sel_key;
  uint64_t sel_sec;
  uint32_t sel_found;
  uint64_t n_cand;
  uint64_t total_len;
  uint32_t cidx_found;
};

// Find digit d of a (group-summed) histogram with above(d) < r <= above(d) + h[d], from
// the top.  Histograms of the whole group are summed through DSMEM.
template <int NT>
__device__ void find_digit(Grp& g, Shared& sh, const uint32_t* H, int nb, uint64_t r, uint32_t* stage = nullptr) {
  const int per = (nb + NT - 1) / NT;
  if (g.size > 1 && stage) {
    // sum the group's histograms into local smem first: independent DSMEM loads, one round trip
    cg::cluster_group cl = cg::this_cluster();
    for (int b = threadIdx.x; b < nb; b += NT) {
      uint32_t v[8];
#pragma unroll
      for (int rr = 0; rr < 8; ++rr) v[rr] = rr < (int)g.size ? *cl.map_shared_rank(H + b, (unsigned)rr) : 0u;
      uint32_t acc = 0;
#pragma unroll
      for (int rr = 0; rr < 8; ++rr) acc += v[rr];
      stage[b] = acc;
    }
    __syncthreads();
    Grp g1 = g;
    g1.size = 1;
    find_digit<NT>(g1, sh, stage, nb, r, nullptr);
    return;
  }
  cg::cluster_group cl = cg::this_cluster();
  auto bin = [&](int b) -> uint64_t {
    if (g.size == 1) return H[b];
    uint64_t v = 0;
    for (uint32_t rr = 0; rr < g.size; ++rr) v += *cl.map_shared_rank(H + b, rr);
    return v;
  };
  uint64_t s = 0;
  for (int k = 0; k < per; ++k) {
    const int b = nb - 1 - (threadIdx.x * per + k);
    if (b >= 0) s += bin(b);
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
      const uint64_t h = bin(b);
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
// fn(bits, idx, &key).  Fallback for huge single-value tie sets.
template <int NT, class KeyFn>
__device__ uint64_t radix_select64(Grp& g, Shared& sh, uint32_t* hist, const List& L, uint32_t n, uint64_t r,
                                   KeyFn fn) {
  const int shifts[6] = {53, 42, 31, 20, 9, 0};
  const int widths[6] = {11, 11, 11, 11, 11, 9};
  uint64_t prefix = 0, mask = 0;
  for (int lev = 0; lev < 6; ++lev) {
    const int shf = shifts[lev], nb = 1 << widths[lev];
    uint32_t* H = hist + (g.size > 1 ? g.hpar * HB : 0);
    g.hpar ^= 1;
    for (int i = threadIdx.x; i < nb; i += NT) H[i] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += NT) {
      uint64_t k;
      if (fn(L.bits(i), L.idx(i), k) && (k & mask) == prefix) atomicAdd(&H[(int)((k >> shf) & (uint64_t)(nb - 1))], 1u);
    }
    g.sync();
    find_digit<NT>(g, sh, H, nb, r, hist + 2 * HB);
    prefix |= (uint64_t)sh.fd_digit << shf;
    mask |= (uint64_t)(nb - 1) << shf;
    r -= sh.fd_above;
    if (g.size == 1) __syncthreads();
  }
  return prefix;
}

// Result of an exact select: the element at 1-based rank r by (key desc, sec asc).
struct SelRes {
  uint32_t key;    // key of the cut element
  uint64_t sec;    // its secondary key (valid unless all_ties)
  uint64_t n_gt;   // elements with key > key
  uint64_t n_eq;   // elements with key == key
  uint64_t r_eq;   // how many of the key == key elements rank at or above the cut
  int all_ties;    // r_eq == n_eq (no secondary test needed)
};

// Exact select.  Levels of 2048-bin histograms narrow [klo, khi) to the bin holding rank
// r; the bin's elements are gathered and ranked exactly by (key desc, sec asc).  If the bin
// is one key value with more than GCAP members, the secondary order is resolved by a radix
// select on the hash, or by the flat-order ordinal for indices.
template <int NT, class Pred, class KeyF, class SecF>
__device__ SelRes select_exact(Grp& g, Shared& sh, uint32_t* scratch, const List& L, uint32_t n, Pred pred,
                               KeyF keyf, SecF secf, uint64_t klo, uint64_t khi, uint64_t r, bool sec_is_idx) {
  constexpr int NW = NT / 32;
  uint32_t* hist = scratch;
  GatE* gl = reinterpret_cast<GatE*>(scratch + 2 * HB);
  GatE* gc = g.size > 1 ? gl + GCAP : gl;
  const int tid = threadIdx.x;
  uint64_t n_gt = 0, cnt = 0;
  for (;;) {
    const uint64_t span = khi - klo;
    const int bl = span > 1 ? 64 - __clzll(span - 1) : 0;
    const int shf = bl > 11 ? bl - 11 : 0;
    const int nb = (int)(((span - 1) >> shf) + 1);
    uint32_t* H = hist + (g.size > 1 ? g.hpar * HB : 0);
    g.hpar ^= 1;
    for (int i = tid; i < nb; i += NT) H[i] = 0;
    __syncthreads();
    list_foreach<NT>(L, n, [&](uint32_t b, uint32_t x) {
      if (pred(b, x)) {
        const uint64_t k = keyf(b);
        if (k >= klo && k < khi) atomicAdd(&H[(int)((k - klo) >> shf)], 1u);
      }
    });
    g.sync();
    find_digit<NT>(g, sh, H, nb, r, reinterpret_cast<uint32_t*>(gc));
    const uint64_t dg = sh.fd_digit;
    n_gt += sh.fd_above;
    r -= sh.fd_above;
    cnt = sh.fd_eq;
    klo = klo + (dg << shf);
    const uint64_t nhi = klo + (1ull << shf);
    khi = nhi < khi ? nhi : khi;
    if (g.size == 1) __syncthreads();
    if (cnt <= GCAP || shf == 0) break;
  }
  SelRes res;
  if (cnt > GCAP) {
    // one key value with a huge tie set (e.g. bf16 or constant tensors)
    res.key = (uint32_t)klo;
    res.n_gt = n_gt;
    res.n_eq = cnt;
    res.r_eq = r;
    res.all_ties = r == cnt;
    res.sec = 0;
    if (!res.all_ties) {
      const uint32_t kk = (uint32_t)klo;
      if (!sec_is_idx) {
        const uint64_t top = radix_select64<NT>(g, sh, hist, L, n, r, [&](uint32_t b, uint32_t x, uint64_t& k) {
          if (!pred(b, x) || keyf(b) != kk) return false;
          k = ~secf(b, x);
          return true;
        });
        res.sec = ~top;
      } else {
        // r-th match in flat order: per-warp counts over contiguous segments, then locate
        const uint32_t seg = (n + NW - 1) / NW;
        const int wid = tid >> 5, lane = tid & 31;
        const uint32_t w0 = wid * seg, w1 = w0 + seg < n ? w0 + seg : n;
        uint32_t c = 0;
        for (uint32_t i = w0 + lane; i < w1; i += 32) c += (pred(L.bits(i), L.idx(i)) && keyf(L.bits(i)) == kk);
        c = __reduce_add_sync(0xFFFFFFFFu, c);
        if (lane == 0) sh.red[wid] = c;
        __syncthreads();
        uint64_t* slot = g.slot();
        if (tid == 0) {
          uint64_t t = 0;
          for (int w = 0; w < NW; ++w) t += sh.red[w];
          slot[0] = t;
          sh.cidx_found = 0;
        }
        g.allsum(1, sh.vec, sh.pre);
        const uint64_t want = r - 1;  // 0-based ordinal among ties, group-wide
        uint64_t base = sh.pre[0];
        for (int w = 0; w < NW; ++w) {
          if (want >= base && want < base + sh.red[w] && wid == w) {
            uint64_t run = base;
            for (uint32_t i0 = w0; i0 < w1; i0 += 32) {
              const uint32_t i = i0 + lane;
              const bool m = i < w1 && pred(L.bits(i), L.idx(i)) && keyf(L.bits(i)) == kk;
              const uint32_t bal = __ballot_sync(0xFFFFFFFFu, m);
              if (m && run + __popc(bal & ((1u << lane) - 1u)) == want) {
                sh.sel_sec = L.idx(i);
                sh.cidx_found = 1;
              }
              run += __popc(bal);
            }
          }
          base += sh.red[w];
        }
        __syncthreads();
        uint64_t* slot2 = g.slot();
        if (tid == 0) slot2[0] = sh.cidx_found ? sh.sel_sec + 1 : 0;
        g.allsum(1, sh.vec, nullptr);
        res.sec = sh.vec[0] - 1;
      }
    }
    return res;
  }
  // gather the bin's elements (unordered) and rank them exactly
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
  const uint32_t m = (uint32_t)cnt;
  if (g.size > 1) {
    g.sync();
    cg::cluster_group cl = cg::this_cluster();
    // concatenate every CTA's gather buffer (rank order) into gc
    uint32_t off = 0;
    for (uint32_t rr = 0; rr < g.size; ++rr) {
      const uint32_t c = *cl.map_shared_rank(&sh.gcount, rr);
      const GatE* src = cl.map_shared_rank(gl, rr);
      for (uint32_t i = tid; i < c; i += NT) gc[off + i] = src[i];
      off += c;
    }
    g.sync();  // peers may now reuse their gather buffers
  } else {
    __syncthreads();
  }
  // rank: element at 0-based position r-1 by (key desc, sec asc)
  if (tid == 0) sh.sel_found = 0;
  __syncthreads();
  if (m <= 256) {
    for (uint32_t i = tid; i < m; i += NT) {
      const uint32_t ki = gc[i].key;
      const uint64_t si = gc[i].sec;
      uint32_t rank = 0;
      for (uint32_t j = 0; j < m; ++j) {
        const uint32_t kj = gc[j].key;
        rank += (kj > ki) || (kj == ki && gc[j].sec < si);
      }
      if (rank == r - 1) {
        sh.sel_key = ki;
        sh.sel_sec = si;
        sh.sel_found = 1;
      }
    }
  } else {
    // bitonic sort (descending key, ascending sec) over the next power of two
    uint32_t p2 = 1;
    while (p2 < m) p2 <<= 1;
    for (uint32_t i = m + tid; i < p2; i += NT) { gc[i].key = 0; gc[i].sec = ~0ull; gc[i].idx = 0; }
    __syncthreads();
    for (uint32_t k = 2; k <= p2; k <<= 1) {
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        for (uint32_t i = tid; i < p2; i += NT) {
          const uint32_t ixj = i ^ j;
          if (ixj > i) {
            const GatE A = gc[i], Bv = gc[ixj];
            const bool a_first = A.key > Bv.key || (A.key == Bv.key && A.sec < Bv.sec);
            const bool up = (i & k) == 0;
            if (up != a_first) { gc[i] = Bv; gc[ixj] = A; }
          }
        }
        __syncthreads();
      }
    }
    if (tid == 0) {
      sh.sel_key = gc[r - 1].key;
      sh.sel_sec = gc[r - 1].sec;
      sh.sel_found = 1;
    }
  }
  __syncthreads();
  const uint32_t ks = sh.sel_key;
  uint32_t gt = 0, eq = 0;
  for (uint32_t i = tid; i < m; i += NT) {
    gt += gc[i].key > ks;
    eq += gc[i].key == ks;
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

template <int DT>
__device__ __forceinline__ uint32_t load_bits(const void* x, uint64_t e) {
  if (DT == SIF_DTYPE_F32) return __ldg(reinterpret_cast<const uint32_t*>(x) + e);
  return (uint32_t)__ldg(reinterpret_cast<const unsigned short*>(x) + e) << 16;
}

// ---------------------------------------------------------------------------------------
// Phase A: stream the slice [s0, s1) once; counts + stable candidate compaction.
struct Counts {
  uint32_t maxkey;
};

// One pass over the slice: max |x| key (NaN/Inf detection, atkf.py:49-51) and the stable
// compaction of candidates (|x| >= lo_p for x >= 0, |x| >= lo_n for x < 0), in flat order.
// Each thread owns 16 contiguous elements per chunk (4 x 128-bit loads for fp32, 2 for
// bf16); the next chunk is prefetched into registers while the current one is compacted.
// ASYM: lambda > 0 thresholds differ by sign.
template <int DT, int NT, bool ASYM>
__device__ __forceinline__ void classify_store(const uint32_t (&v)[16], uint32_t valid, uint32_t e0, uint32_t lo_p,
                                               uint32_t lo_n, const List& L, uint32_t* scan, uint32_t& ncand,
                                               uint32_t& mk) {
  uint32_t m = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const uint32_t key = v[j] & 0x7FFFFFFFu;
    const bool in = (valid >> j) & 1u;
    mk = max(mk, in ? key : 0u);
    const uint32_t thr = ASYM ? ((v[j] >> 31) ? lo_n : lo_p) : lo_p;
    m |= (in && key >= thr) ? (1u << j) : 0u;
  }
  uint32_t tot;
  const uint32_t ex = block_excl_scan_u32(__popc(m), scan, &tot);
  uint32_t off = ncand + ex;
  if (ncand + tot <= L.cap) {
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if ((m >> j) & 1u) { L.sb[off] = v[j]; L.si[off] = e0 + j; ++off; }
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if ((m >> j) & 1u) { L.set(off, v[j], e0 + j); ++off; }
  }
  ncand += tot;
}

template <int DT>
__device__ __forceinline__ void load16(const void* x, uint32_t e, uint32_t (&v)[16]) {
  if (DT == SIF_DTYPE_F32) {
    const uint4* p = reinterpret_cast<const uint4*>(reinterpret_cast<const uint32_t*>(x) + e);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint4 q = __ldcs(p + k);
      v[4 * k] = q.x; v[4 * k + 1] = q.y; v[4 * k + 2] = q.z; v[4 * k + 3] = q.w;
    }
  } else {
    const uint4* p = reinterpret_cast<const uint4*>(reinterpret_cast<const unsigned short*>(x) + e);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const uint4 q = __ldcs(p + k);
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) { v[8 * k + 2 * i] = w[i] << 16; v[8 * k + 2 * i + 1] = w[i] & 0xFFFF0000u; }
    }
  }
}

template <int DT, int NT, bool ASYM>
__device__ __noinline__ void stream_pass_t(const void* x, uint32_t s0, uint32_t s1, uint32_t lo_p, uint32_t lo_n,
                                           const List L, Shared& sh, Counts& c) {
  const uint32_t tid = threadIdx.x;
  uint32_t* scan = reinterpret_cast<uint32_t*>(sh.scan);
  const uint32_t a0 = min(s1, (s0 + 15u) & ~15u), a1 = max(a0, s1 & ~15u);
  uint32_t ncand = 0, mk = 0;
  uint32_t v[16];
  // ragged head [s0, a0): at most 15 elements, one per thread (flat order kept)
  if (a0 > s0) {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = 0;
    const uint32_t e = s0 + tid;
    uint32_t valid = 0;
    if (e < a0) { v[0] = load_bits<DT>(x, e); valid = 1; }
    classify_store<DT, NT, ASYM>(v, valid, e, lo_p, lo_n, L, scan, ncand, mk);
  }
  const uint32_t CH = NT * 16u;
  uint32_t nx[16];
  if (a0 < a1 && a0 + tid * 16u < a1) load16<DT>(x, a0 + tid * 16u, v);
  for (uint32_t base = a0; base < a1; base += CH) {
    const uint32_t e = base + tid * 16u;
    const uint32_t en = e + CH;
    const bool more = base + CH < a1;
    if (more && en < a1) load16<DT>(x, en, nx);
    classify_store<DT, NT, ASYM>(v, e < a1 ? 0xFFFFu : 0u, e, lo_p, lo_n, L, scan, ncand, mk);
    if (more) {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = nx[j];
    }
  }
  // ragged tail [a1, s1)
  if (s1 > a1) {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = 0;
    const uint32_t e = a1 + tid;
    uint32_t valid = 0;
    if (e < s1) { v[0] = load_bits<DT>(x, e); valid = 1; }
    classify_store<DT, NT, ASYM>(v, valid, e, lo_p, lo_n, L, scan, ncand, mk);
  }
  c.maxkey = mk;
  if (tid == 0) sh.n_cand = ncand;
  __syncthreads();
}

template <int DT, int NT>
__device__ __forceinline__ void stream_pass(const void* x, uint64_t T, uint64_t s0, uint64_t s1, uint32_t lo_p,
                                            uint32_t lo_n, const List& L, Shared& sh, Counts& c) {
  (void)T;
  if (lo_p != lo_n) stream_pass_t<DT, NT, true>(x, (uint32_t)s0, (uint32_t)s1, lo_p, lo_n, L, sh, c);
  else stream_pass_t<DT, NT, false>(x, (uint32_t)s0, (uint32_t)s1, lo_p, lo_n, L, sh, c);
}

// Group-reduce the stream pass: candidate total and max |x| key.
template <int NT>
__device__ void reduce_counts(Grp& g, Shared& sh, Counts& c) {
  uint64_t* slot = g.slot();
  if (threadIdx.x < 2) slot[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t mk = __reduce_max_sync(0xFFFFFFFFu, c.maxkey);
  if ((threadIdx.x & 31) == 0) atomicMax((unsigned long long*)&slot[1], (unsigned long long)mk);
  if (threadIdx.x == 0) slot[0] = sh.n_cand;
  g.allsum(1, sh.vec, nullptr);
  uint64_t* prev = g.slots + (g.parity ^ 1) * 64;  // this CTA's slot (still intact)
  uint64_t m = 0;
  if (g.size == 1) m = prev[1];
  else {
    cg::cluster_group cl = cg::this_cluster();
    for (uint32_t r = 0; r < g.size; ++r) {
      const uint64_t y = *cl.map_shared_rank(prev + 1, r);
      m = y > m ? y : m;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) sh.vec[1] = m;
  __syncthreads();
}

// Count candidates with key >= lo and key >= hi (group totals).
template <int NT>
__device__ void count_ge(Grp& g, Shared& sh, const List& L, uint32_t n, uint32_t lo, uint32_t hi, uint64_t* clo,
                         uint64_t* chi) {
  uint32_t a = 0, b = 0;
  list_foreach<NT>(L, n, [&](uint32_t bits, uint32_t) {
    const uint32_t k = bits & 0x7FFFFFFFu;
    a += k >= lo;
    b += k >= hi;
  });
  a = __reduce_add_sync(0xFFFFFFFFu, a);
  b = __reduce_add_sync(0xFFFFFFFFu, b);
  uint64_t* slot = g.slot();
  if (threadIdx.x < 2) slot[threadIdx.x] = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    atomicAdd((unsigned long long*)&slot[0], (unsigned long long)a);
    atomicAdd((unsigned long long*)&slot[1], (unsigned long long)b);
  }
  g.allsum(2, sh.vec, nullptr);
  *clo = sh.vec[0];
  *chi = sh.vec[1];
  __syncthreads();
}

// ---------------------------------------------------------------------------------------
// Per-IF encoder state, kept in shared memory so each phase (a separate, non-inlined
// function) starts with a small live register set instead of one huge allocation.
struct Ctx {
  const void* x;
  uint8_t* out;
  uint64_t out_cap, seed;
  uint32_t N, K, dtype, cb;
  uint64_t T, s0, s1, kk;
  FastDiv fk;
  double s, lam, delta;
  int m_plus, m_minus, q_bit, mode, atkf_only, maxb, ifi;
  const uint8_t* fixed_q;
  uint64_t* prof;
  uint32_t* t4;
  uint32_t* scratch;
  uint64_t *b_sum, *b_pre, *b_N, *b_off;
  double *b_o64, *b_inv;
  uint32_t *b_n, *b_rs, *b_min, *b_max, *b_q, *b_act, *cut_key, *cut_idx, *wcnt, *woff;
  List L;
  Perm M;
  uint32_t lo, hi, lo_neg, maxkey, tau_key, ncand, nkept;
  uint64_t cnt_nz, cnt_lo, cnt_hi, ck_star, h_star, kept_pre;
  double tau, tau_p, tau_m;
  int zero_mode, only_nonzero, keep_none, use_cls, tie_all, nonfinite;
  uint64_t cnt_sign[2], meff[2], base[2];
  uint32_t kmin[2], kmax[2];
  int B, ncut0, ncut;
  uint64_t P;
};

__device__ __forceinline__ void phase_mark(const Ctx& c, const Grp& g, int k) {
  if (c.prof && g.rank == 0 && threadIdx.x == 0) c.prof[(uint64_t)c.ifi * 32 + k] = gtimer();
}

// ---- Phase S: sampled bracket [lo, hi) for tau (identical in every CTA of the group)
template <int DT, int NT>
__device__ __noinline__ Grp phase_sample(Ctx& c, Grp g, Shared& sh) {
  const int tid = threadIdx.x;
  const uint64_t T = c.T, kk = c.kk;
  uint32_t lo = 1, hi = kInfKey;
  if (T > 32768 && kk > 0 && 2 * kk <= T) {
    constexpr int NSECT = 512, SB = 8192;  // 512 sectors x 8 elements; 13-bit key bins
    constexpr int PERT = (NSECT + NT - 1) / NT;
    uint32_t* sh8k = c.scratch;
    for (int i = tid; i < SB; i += NT) sh8k[i] = 0;
    uint32_t sv[PERT][8];
#pragma unroll
    for (int k = 0; k < PERT; ++k) {
      const int j = tid + k * NT;
#pragma unroll
      for (int q = 0; q < 8; ++q) sv[k][q] = 0;
      if (j < NSECT) {
        // low-discrepancy (Weyl) sector positions avoid aliasing with row structure
        const uint64_t nsec = T / 8;
        const uint64_t frac = (uint64_t)(uint32_t)((uint32_t)j * 0x9E3779B9u);  // j * golden ratio mod 1
        const uint64_t e = ((frac * nsec) >> 32) * 8;
        if (DT == SIF_DTYPE_F32) {
          const uint4* q4 = reinterpret_cast<const uint4*>(reinterpret_cast<const uint32_t*>(c.x) + e);
          const uint4 v0 = __ldg(q4), v1 = __ldg(q4 + 1);
          sv[k][0] = v0.x; sv[k][1] = v0.y; sv[k][2] = v0.z; sv[k][3] = v0.w;
          sv[k][4] = v1.x; sv[k][5] = v1.y; sv[k][6] = v1.z; sv[k][7] = v1.w;
        } else {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const unsigned short*>(c.x) + e));
          const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) { sv[k][2 * q] = w[q] << 16; sv[k][2 * q + 1] = w[q] & 0xFFFF0000u; }
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < PERT; ++k) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t key = sv[k][q] & 0x7FFFFFFFu;
        if (key && key < kNonFiniteKey) atomicAdd(&sh8k[key >> 18], 1u);
      }
    }
    __syncthreads();
    const double S = NSECT * 8.0;
    const double qf = (double)kk / (double)T;
    const double sd = sqrt(qf * (1.0 - qf) * S);
    const double rlo = ceil(qf * S + 3.0 * sd + 2.0);
    const double rhi = floor(qf * S - 3.0 * sd - 2.0);
    Grp g1 = g;
    g1.size = 1;
    find_digit<NT>(g1, sh, sh8k, SB, (uint64_t)rlo);
    const bool lo_ok = sh.fd_found != 0;
    const uint32_t lo_b = sh.fd_digit;
    bool hi_ok = false;
    uint32_t hi_b = 0;
    if (rhi >= 1.0) {
      find_digit<NT>(g1, sh, sh8k, SB, (uint64_t)rhi);
      hi_ok = sh.fd_found != 0;
      hi_b = sh.fd_digit;
    }
    lo = lo_ok ? (lo_b << 18) : 1u;
    if (lo == 0) lo = 1;
    hi = (hi_ok && hi_b + 1u < (uint32_t)SB) ? ((hi_b + 1u) << 18) : kInfKey;
  }
  uint32_t lo_neg = lo;
  if (c.lam > 0.0 && lo > 1) {
    const double t = __dmul_rn(__dsub_rn(1.0, c.lam), (double)__uint_as_float(lo));
    const uint32_t k2 = __float_as_uint(__double2float_rd(t));
    lo_neg = k2 > 1 ? k2 : 1u;
  }
  __syncthreads();
  if (tid == 0) { c.lo = lo; c.hi = hi; c.lo_neg = lo_neg; }
  __syncthreads();
  return g;
}

// ---- Phase A: stream the slice, count, compact candidates (+ fallback re-stream)
template <int DT, int NT>
__device__ __noinline__ Grp phase_stream(Ctx& c, Grp g, Shared& sh) {
  const int tid = threadIdx.x;
  const uint64_t kk = c.kk;
  uint32_t lo = c.lo, hi = c.hi, lo_neg = c.lo_neg;
  Counts k;
  stream_pass<DT, NT>(c.x, c.T, c.s0, c.s1, lo, lo_neg, c.L, sh, k);
  reduce_counts<NT>(g, sh, k);
  uint32_t maxkey = (uint32_t)sh.vec[1];
  const int nonfinite = maxkey >= kNonFiniteKey;
  uint64_t cnt_lo = 0, cnt_hi = 0;
  if (!nonfinite) count_ge<NT>(g, sh, c.L, (uint32_t)sh.n_cand, lo, hi, &cnt_lo, &cnt_hi);
  uint64_t cnt_nz = cnt_lo;  // exact when lo <= 1, else a lower bound (only compared with kk)
  if (!nonfinite && kk > 0 && cnt_lo < kk && lo > (c.atkf_only ? 0u : 1u)) {
    // bracket missed (or tau == 0): re-stream keeping every nonzero (every element in
    // ATKF-only mode)
    const uint32_t new_hi = lo;
    lo = c.atkf_only ? 0u : 1u;
    lo_neg = lo;
    hi = new_hi;
    stream_pass<DT, NT>(c.x, c.T, c.s0, c.s1, lo, lo_neg, c.L, sh, k);
    reduce_counts<NT>(g, sh, k);
    maxkey = (uint32_t)sh.vec[1];
    count_ge<NT>(g, sh, c.L, (uint32_t)sh.n_cand, 1u, hi, &cnt_nz, &cnt_hi);
    cnt_lo = cnt_nz;
  }
  __syncthreads();
  if (tid == 0) {
    c.lo = lo; c.hi = hi; c.lo_neg = lo_neg;
    c.cnt_nz = cnt_nz; c.cnt_lo = cnt_lo; c.cnt_hi = cnt_hi;
    c.maxkey = maxkey;
    c.nonfinite = nonfinite;
    c.zero_mode = kk > 0 && lo == 0;
    c.ncand = (uint32_t)sh.n_cand;
  }
  __syncthreads();
  return g;
}

// ---- Phase B: tau, class (lambda > 0) and the tie cut (atkf.py:71-84)
template <int NT>
__device__ __noinline__ Grp phase_select(Ctx& c, Grp g, Shared& sh) {
  const int tid = threadIdx.x;
  const uint64_t kk = c.kk, seed = c.seed;
  const uint64_t cnt_nz = c.cnt_nz, cnt_hi = c.cnt_hi;
  const uint32_t lo = c.lo, hi = c.hi, maxkey = c.maxkey, ncand = c.ncand;
  const bool zero_mode = c.zero_mode != 0;
  const List L = c.L;
  auto hash_of = [seed](uint32_t, uint32_t x) -> uint64_t { return splitmix(seed, x); };
  auto key31 = [](uint32_t b) -> uint64_t { return b & 0x7FFFFFFFu; };
  auto all_pred = [](uint32_t, uint32_t) { return true; };
  uint32_t tau_key = 0;
  uint64_t ck_star = 0, h_star = 0;
  bool tie_all = true;
  const bool keep_none = kk == 0;
  const bool only_nonzero = kk > 0 && cnt_nz < kk && !zero_mode;  // tau == 0 in payload mode
  if (kk > 0 && !only_nonzero) {
    if (zero_mode && cnt_nz < kk) {
      // tau == 0 (ATKF-only mode): every nonzero is kept; choose kk - nnz zeros by hash
      const SelRes s = select_exact<NT>(g, sh, c.scratch, L, ncand, all_pred, key31, hash_of, 0, 1, kk - cnt_nz, false);
      h_star = s.sec;
      tie_all = s.all_ties;
    } else {
      uint64_t ra, rb, r;
      if (cnt_hi >= kk || hi == kInfKey) { ra = (hi == kInfKey ? lo : hi); rb = (uint64_t)maxkey + 1; r = kk; }
      else { ra = lo; rb = hi; r = kk - cnt_hi; }
      const SelRes s = select_exact<NT>(g, sh, c.scratch, L, ncand, all_pred, key31, hash_of, ra, rb, r, false);
      tau_key = s.key;
      ck_star = s.key;
      h_star = s.sec;
      tie_all = s.all_ties;
    }
  }
  const double tau = kk > 0 ? (double)__uint_as_float(tau_key) : (double)__uint_as_float(maxkey);
  const double tau_p = __dmul_rn(__dadd_rn(1.0, c.lam), tau);
  const double tau_m = -__dmul_rn(__dsub_rn(1.0, c.lam), tau);
  const bool use_cls = c.lam > 0.0 && kk > 0 && !only_nonzero;
  if (use_cls) {
    // composite key (strict << 31 | |x|) selects class, magnitude and ties at once
    auto ckey = [tau_p, tau_m](uint32_t b) -> uint64_t {
      const double v = (double)__uint_as_float(b);
      return ((v > tau_p || v < tau_m) ? (1ull << 31) : 0ull) | (uint64_t)(b & 0x7FFFFFFFu);
    };
    const SelRes s = select_exact<NT>(g, sh, c.scratch, L, ncand, all_pred, ckey, hash_of, 0, 1ull << 32, kk, false);
    ck_star = s.key;
    h_star = s.sec;
    tie_all = s.all_ties;
  }
  __syncthreads();
  if (tid == 0) {
    c.tau_key = tau_key; c.ck_star = ck_star; c.h_star = h_star; c.tie_all = tie_all;
    c.keep_none = keep_none; c.only_nonzero = only_nonzero; c.use_cls = use_cls;
    c.tau = tau; c.tau_p = tau_p; c.tau_m = tau_m;
  }
  __syncthreads();
  return g;
}

// ---- Phase C: kept set, stable in-place compaction (8 elements per thread per chunk)
template <int NT>
__device__ __noinline__ Grp phase_kept(Ctx& c, Grp g, Shared& sh) {
  const int tid = threadIdx.x, lane = tid & 31;
  const List L = c.L;
  const uint32_t ncand = c.ncand;
  const bool keep_none = c.keep_none, only_nonzero = c.only_nonzero, zero_mode = c.zero_mode;
  const bool use_cls = c.use_cls, tie_all = c.tie_all;
  const uint64_t ck_star = c.ck_star, h_star = c.h_star, seed = c.seed;
  const double tau_p = c.tau_p, tau_m = c.tau_m;
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
  constexpr int E = 8;
  uint32_t run = 0;
  uint64_t sp = 0, sm = 0;
  uint32_t mn0 = 0x7FFFFFFFu, mn1 = 0x7FFFFFFFu, mx0 = 0, mx1 = 0;
  for (uint32_t base = 0; base < ncand; base += NT * E) {
    uint32_t bb[E], xx[E];
    uint32_t km = 0;
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const uint32_t i = base + tid * E + j;
      bb[j] = 0;
      xx[j] = 0;
      if (i < ncand) {
        bb[j] = L.bits(i);
        xx[j] = L.idx(i);
        if (kept_of(bb[j], xx[j])) km |= 1u << j;
      }
    }
    uint64_t tot;
    const uint64_t ex = block_excl_scan_u64((uint64_t)__popc(km), sh.scan, &tot);
    uint32_t o = run + (uint32_t)ex;
#pragma unroll
    for (int j = 0; j < E; ++j) {
      if (km & (1u << j)) {
        L.set(o++, bb[j], xx[j]);
        const uint32_t kj = bb[j] & 0x7FFFFFFFu;
        if (kj != 0) {
          if (bb[j] >> 31) { ++sm; mn1 = kj < mn1 ? kj : mn1; mx1 = kj > mx1 ? kj : mx1; }
          else { ++sp; mn0 = kj < mn0 ? kj : mn0; mx0 = kj > mx0 ? kj : mx0; }
        }
      }
    }
    run += (uint32_t)tot;
  }
  sp = warp_sum_u64(sp);
  sm = warp_sum_u64(sm);
  mn0 = __reduce_min_sync(0xFFFFFFFFu, mn0);
  mn1 = __reduce_min_sync(0xFFFFFFFFu, mn1);
  mx0 = __reduce_max_sync(0xFFFFFFFFu, mx0);
  mx1 = __reduce_max_sync(0xFFFFFFFFu, mx1);
  uint64_t* slot = g.slot();
  if (tid < 7) slot[tid] = tid >= 3 && tid < 5 ? 0x7FFFFFFFull : 0ull;
  __syncthreads();
  if (lane == 0) {
    atomicAdd((unsigned long long*)&slot[0], (unsigned long long)sp);
    atomicAdd((unsigned long long*)&slot[1], (unsigned long long)sm);
    atomicMin((unsigned long long*)&slot[3], (unsigned long long)mn0);
    atomicMin((unsigned long long*)&slot[4], (unsigned long long)mn1);
    atomicMax((unsigned long long*)&slot[5], (unsigned long long)mx0);
    atomicMax((unsigned long long*)&slot[6], (unsigned long long)mx1);
  }
  if (tid == 0) slot[2] = run;
  g.allsum(3, sh.vec, sh.pre);
  uint64_t* prev = g.slots + (g.parity ^ 1) * 64;
  uint64_t k0 = 0x7FFFFFFF, k1 = 0x7FFFFFFF, k2 = 0, k3 = 0;
  {
    cg::cluster_group cl = cg::this_cluster();
    for (uint32_t r = 0; r < g.size; ++r) {
      const uint64_t* q = g.size == 1 ? prev : cl.map_shared_rank(prev, r);
      k0 = q[3] < k0 ? q[3] : k0;
      k1 = q[4] < k1 ? q[4] : k1;
      k2 = q[5] > k2 ? q[5] : k2;
      k3 = q[6] > k3 ? q[6] : k3;
    }
  }
  __syncthreads();
  if (tid == 0) {
    c.nkept = run;
    c.cnt_sign[0] = sh.vec[0];
    c.cnt_sign[1] = sh.vec[1];
    c.kept_pre = sh.pre[2];
    c.kmin[0] = (uint32_t)k0;
    c.kmax[0] = (uint32_t)k2;
    c.kmin[1] = (uint32_t)k1;
    c.kmax[1] = (uint32_t)k3;
  }
  __syncthreads();
  return g;
}

// ---- Phase D: MS cut elements (msplit.py:54-80), value desc then flat idx asc
template <int NT>
__device__ __noinline__ Grp phase_cuts(Ctx& c, Grp g, Shared& sh) {
  const int tid = threadIdx.x;
  const int mcfg[2] = {c.m_plus, c.m_minus};
  uint64_t meff[2], base[2];
  for (int s = 0; s < 2; ++s) {
    const uint64_t nz = c.cnt_sign[s], m = (uint64_t)mcfg[s];
    meff[s] = nz < m ? nz : m;
    if (meff[s] < 1) meff[s] = 1;
    base[s] = nz / meff[s];
  }
  const int B = (int)(meff[0] + meff[1]);
  const int ncut0 = (int)meff[0] - 1;
  const int ncut = B - 2;
  const List L = c.L;
  const uint32_t nkept = c.nkept;
  for (int ci = 0; ci < ncut; ++ci) {
    const uint32_t s = ci < ncut0 ? 0u : 1u;
    const int j = (s == 0 ? ci : ci - ncut0) + 1;
    const uint64_t rank0 = (uint64_t)j * base[s];
    const uint64_t klo = c.kmin[s], khi = (uint64_t)c.kmax[s] + 1;
    const SelRes r = select_exact<NT>(g, sh, c.scratch, L, nkept, [s](uint32_t b, uint32_t) { return (b >> 31) == s; },
                                      [](uint32_t b) -> uint64_t { return b & 0x7FFFFFFFu; },
                                      [](uint32_t, uint32_t x) -> uint64_t { return x; }, klo, khi > klo ? khi : klo + 1,
                                      rank0 + 1, true);
    if (tid == 0) {
      c.cut_key[ci] = r.key;
      c.cut_idx[ci] = (uint32_t)r.sec;
    }
    __syncthreads();
  }
  if (tid == 0) {
    c.meff[0] = meff[0]; c.meff[1] = meff[1]; c.base[0] = base[0]; c.base[1] = base[1];
    c.B = B; c.ncut0 = ncut0; c.ncut = ncut;
  }
  __syncthreads();
  return g;
}

__device__ __forceinline__ int block_of(const uint32_t* cut_key, const uint32_t* cut_idx, int ncut0, int ncut,
                                        int meff0, uint32_t b, uint32_t x) {
  const uint32_t key = b & 0x7FFFFFFFu;
  const int s = (int)(b >> 31);
  const int c0 = s ? ncut0 : 0, cn = s ? ncut : ncut0;
  int blk = 0;
  for (int cc = c0; cc < cn; ++cc) {
    const uint32_t k2 = cut_key[cc];
    if (key < k2 || (key == k2 && x >= cut_idx[cc])) ++blk;
    else break;
  }
  return (s ? meff0 : 0) + blk;
}

// ---- Phase E: members per block in flat (CSR) order: warp-segmented stable walk.
// Block ids (B <= 8) are one-hot encoded in 8-bit fields of a u64; one warp inclusive
// scan gives every lane its rank among same-block lanes and the warp's per-block totals.
// Lane b keeps the running count of block b in a register.  B > 8 uses match_any.
__device__ __forceinline__ uint64_t warp_incl_scan_u64(uint64_t x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

template <int NT>
__device__ __noinline__ Grp phase_members(Ctx& c, Grp g, Shared& sh, int scratch_bytes) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const List L = c.L;
  const Perm M = c.M;
  const uint32_t nkept = c.nkept;
  const int B = c.B, maxb = c.maxb, ncut0 = c.ncut0, ncut = c.ncut, meff0 = (int)c.meff[0];
  const uint32_t* cut_key = c.cut_key;
  const uint32_t* cut_idx = c.cut_idx;
  uint32_t* wcnt = c.wcnt;
  uint32_t* woff = c.woff;
  uint8_t* bid = reinterpret_cast<uint8_t*>(c.scratch);
  const bool keep_bid = nkept <= (uint32_t)scratch_bytes && B <= 255;
  const bool few = B <= 8;
  const uint32_t lt = (1u << lane) - 1u;
  const uint32_t seg = (nkept + NW - 1) / NW;
  const uint32_t w0 = wid * seg, w1 = (w0 + seg < nkept) ? w0 + seg : nkept;
  // cuts in registers (up to 4 per sign on the fast path)
  uint32_t ck[8], cx[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) { ck[k] = 0; cx[k] = 0; }
  const bool reg_cuts = ncut0 <= 4 && ncut - ncut0 <= 4;
  if (reg_cuts) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k < ncut0) { ck[k] = cut_key[k]; cx[k] = cut_idx[k]; }
      if (k < ncut - ncut0) { ck[4 + k] = cut_key[ncut0 + k]; cx[4 + k] = cut_idx[ncut0 + k]; }
    }
  }
  const int nc1 = ncut - ncut0;
  auto blk_of = [&](uint32_t b, uint32_t x) -> int {
    if (!reg_cuts) return block_of(cut_key, cut_idx, ncut0, ncut, meff0, b, x);
    const uint32_t key = b & 0x7FFFFFFFu;
    const bool neg = (b >> 31) != 0;
    int blk = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t k2 = neg ? ck[4 + k] : ck[k], x2 = neg ? cx[4 + k] : cx[k];
      const bool act = k < (neg ? nc1 : ncut0);
      blk += (act && (key < k2 || (key == k2 && x >= x2))) ? 1 : 0;
    }
    return (neg ? meff0 : 0) + blk;
  };
  // ---- walk 1: block ids and per-warp block counts
  uint32_t run = 0;  // lane b: running count of block b (few) in this warp
  for (int b = lane; b < B; b += 32) wcnt[wid * maxb + b] = 0;
  __syncwarp();
  for (uint32_t i = w0; i < w1; i += 32) {
    const uint32_t e = i + lane;
    const int blk = e < w1 ? blk_of(L.bits(e), L.idx(e)) : -1;
    if (keep_bid && e < w1) bid[e] = (uint8_t)blk;
    if (few) {
      const uint64_t oh = blk >= 0 ? (1ull << (8 * blk)) : 0ull;
      const uint64_t sc = warp_incl_scan_u64(oh);
      const uint64_t tot = __shfl_sync(0xFFFFFFFFu, sc, 31);
      if (lane < B) run += (uint32_t)((tot >> (8 * lane)) & 0xFFull);
    } else {
      const uint32_t peers = __match_any_sync(0xFFFFFFFFu, blk);
      if (blk >= 0 && lane == __ffs(peers) - 1) wcnt[wid * maxb + blk] += __popc(peers);
      __syncwarp();
    }
  }
  if (few && lane < B) wcnt[wid * maxb + lane] = run;
  __syncthreads();
  for (int b = tid; b < B; b += NT) {
    uint32_t acc = 0;
    for (int w = 0; w < NW; ++w) {
      woff[w * maxb + b] = acc;
      acc += wcnt[w * maxb + b];
    }
    c.b_n[b] = acc;
  }
  __syncthreads();
  if (tid == 0) {
    uint32_t acc = 0;
    for (int b = 0; b < B; ++b) { c.b_rs[b] = acc; acc += c.b_n[b]; }
  }
  __syncthreads();
  for (int k = tid; k < NW * B; k += NT) {
    const int w = k / B, b = k - w * B;
    woff[w * maxb + b] += c.b_rs[b];
  }
  __syncthreads();
  // ---- walk 2: stable positions
  uint32_t pos = few && lane < B ? woff[wid * maxb + lane] : 0u;  // lane b: next position of block b
  for (uint32_t i = w0; i < w1; i += 32) {
    const uint32_t e = i + lane;
    int blk = -1;
    if (e < w1) blk = keep_bid ? (int)bid[e] : blk_of(L.bits(e), L.idx(e));
    if (few) {
      const uint64_t oh = blk >= 0 ? (1ull << (8 * blk)) : 0ull;
      const uint64_t sc = warp_incl_scan_u64(oh);
      const uint64_t tot = __shfl_sync(0xFFFFFFFFu, sc, 31);
      const uint32_t basep = __shfl_sync(0xFFFFFFFFu, pos, blk >= 0 ? blk : 0);
      if (blk >= 0) M.set(basep + (uint32_t)((sc >> (8 * blk)) & 0xFFull) - 1u, e);
      if (lane < B) pos += (uint32_t)((tot >> (8 * lane)) & 0xFFull);
    } else {
      const uint32_t peers = __match_any_sync(0xFFFFFFFFu, blk);
      if (blk >= 0) M.set(woff[wid * maxb + blk] + __popc(peers & lt), e);
      __syncwarp();
      if (blk >= 0 && lane == __ffs(peers) - 1) woff[wid * maxb + blk] += __popc(peers);
      __syncwarp();
    }
  }
  __syncthreads();
  for (int b0 = 0; b0 < B; b0 += 64) {
    const int nb = B - b0 < 64 ? B - b0 : 64;
    uint64_t* slot = g.slot();
    if (tid < nb) slot[tid] = c.b_n[b0 + tid];
    g.allsum(nb, sh.vec, sh.pre);
    if (tid < nb) { c.b_N[b0 + tid] = sh.vec[tid]; c.b_pre[b0 + tid] = sh.pre[tid]; }
    __syncthreads();
  }
  return g;
}

// ---- Phase F: block min / max keys (quant.py:50-51)
template <int NT>
__device__ __noinline__ Grp phase_minmax(Ctx& c, Grp g, Shared& sh) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int B = c.B;
  const List L = c.L;
  const Perm M = c.M;
  uint32_t* b_min = c.b_min;
  uint32_t* b_max = c.b_max;
  for (int b = tid; b < B; b += NT) { b_min[b] = 0x7FFFFFFFu; b_max[b] = 0u; }
  __syncthreads();
  for (int b = 0; b < B; ++b) {
    uint32_t mn = 0x7FFFFFFFu, mx = 0;
    const uint32_t rs = c.b_rs[b], n = c.b_n[b];
    for (uint32_t i = tid; i < n; i += NT) {
      const uint32_t k = L.bits(M.get(rs + i)) & 0x7FFFFFFFu;
      mn = k < mn ? k : mn;
      mx = k > mx ? k : mx;
    }
    mn = __reduce_min_sync(0xFFFFFFFFu, mn);
    mx = __reduce_max_sync(0xFFFFFFFFu, mx);
    if (lane == 0) { atomicMin(&b_min[b], mn); atomicMax(&b_max[b], mx); }
  }
  __syncthreads();
  if (g.size > 1) {
    for (int b0 = 0; b0 < B; b0 += 64) {
      const int nb = B - b0 < 64 ? B - b0 : 64;
      uint64_t* my = g.slot();
      if (tid < nb) my[tid] = ((uint64_t)(0x7FFFFFFFu - b_min[b0 + tid]) << 32) | b_max[b0 + tid];
      g.sync();
      cg::cluster_group cl = cg::this_cluster();
      if (tid < nb) {
        uint32_t mn = 0x7FFFFFFFu, mx = 0;
        for (uint32_t r = 0; r < g.size; ++r) {
          const uint64_t v = *cl.map_shared_rank(my + tid, r);
          const uint32_t m0 = 0x7FFFFFFFu - (uint32_t)(v >> 32), m1 = (uint32_t)v;
          mn = m0 < mn ? m0 : mn;
          mx = m1 > mx ? m1 : mx;
        }
        b_min[b0 + tid] = mn;
        b_max[b0 + tid] = mx;
      }
      g.parity ^= 1;
      __syncthreads();
    }
  }
  return g;
}

// ---- Phase G: ABQ (quant.py:102-115) / fixed Q (codec.py:180-181, :194-200)
template <int NT>
__device__ __noinline__ Grp phase_abq(Ctx& c, Grp g, Shared& sh) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int B = c.B, meff0 = (int)c.meff[0], q_bit = c.q_bit;
  const List L = c.L;
  const Perm M = c.M;
  for (int b = tid; b < B; b += NT) {
    const int s = b < meff0 ? 0 : 1;
    const int j = s ? b - meff0 : b;
    const bool empty = c.b_N[b] == 0;
    const bool degen = !empty && c.b_min[b] == c.b_max[b];
    uint32_t q;
    if (c.mode == SIF_MODE_FIXED) q = c.fixed_q[(s ? c.m_plus : 0) + j];
    else if (empty) q = (uint32_t)q_bit;
    else if (degen) q = 1;
    else q = 0;  // searched below
    c.b_act[b] = q == 0 ? 1u : 0u;
    c.b_q[b] = q == 0 ? (uint32_t)q_bit : q;
  }
  __syncthreads();
  if (c.mode != SIF_MODE_FIXED) {
    const uint32_t lref = (1u << q_bit) - 1u;
    const double delta = c.delta;
    for (int q = q_bit - 1; q >= 1; --q) {
      int any = 0;
      for (int b = 0; b < B; ++b) any |= (int)c.b_act[b];
      if (!any) break;
      const uint32_t lv = (1u << q) - 1u;
      const int shift = q_bit - q;
      for (int b = 0; b < B; ++b) {
        if (!c.b_act[b]) continue;
        const double vmin = (double)__uint_as_float(c.b_min[b]), vmax = (double)__uint_as_float(c.b_max[b]);
        const double rng = __dsub_rn(vmax, vmin);
        const double orf = __ddiv_rn(rng, (double)lref), oq = __ddiv_rn(rng, (double)lv);
        const double irf = __drcp_rn(orf), iq = __drcp_rn(oq);
        const uint32_t rs = c.b_rs[b], n = c.b_n[b];
        uint32_t acc = 0;
        for (uint32_t i = tid; i < n; i += NT) {
          const uint32_t k = L.bits(M.get(rs + i)) & 0x7FFFFFFFu;
          const uint32_t cr = quant_code(k, vmin, orf, irf, lref) >> shift;
          const uint32_t cq = quant_code(k, vmin, oq, iq, lv);
          acc += cr > cq ? cr - cq : cq - cr;
        }
        acc = __reduce_add_sync(0xFFFFFFFFu, acc);
        if (lane == 0) sh.red[wid] = acc;
        __syncthreads();
        if (tid == 0) {
          uint64_t t = 0;
          for (int w = 0; w < NW; ++w) t += sh.red[w];
          c.b_sum[b] = t;
        }
        __syncthreads();
      }
      for (int b0 = 0; b0 < B; b0 += 64) {
        const int nb = B - b0 < 64 ? B - b0 : 64;
        uint64_t* slot = g.slot();
        if (tid < nb) slot[tid] = c.b_act[b0 + tid] ? c.b_sum[b0 + tid] : 0ull;
        g.allsum(nb, sh.vec, nullptr);
        if (tid < nb) {
          const int b = b0 + tid;
          if (c.b_act[b]) {
            const double ds = __ddiv_rn((double)sh.vec[tid], (double)c.b_N[b]);
            if (ds > delta) c.b_act[b] = 0;  // first violation stops the descent
            else { c.b_q[b] = (uint32_t)q; if (q == 1) c.b_act[b] = 0; }
          }
        }
        __syncthreads();
      }
    }
  }
  return g;
}

// ---- Phase H: layout (codec.py:269-280), codes in place, zero fill
template <int NT>
__device__ __noinline__ Grp phase_layout(Ctx& c, Grp g, Shared& sh) {
  const int tid = threadIdx.x;
  const int B = c.B;
  if (tid == 0) {
    uint64_t pos = kHeaderBytes + (c.mode == SIF_MODE_FIXED ? (uint64_t)B : 0ull);
    for (int b = 0; b < B; ++b) {
      c.b_off[4 * b + 0] = pos;
      c.b_off[4 * b + 1] = pos + kBlockMetaBytes;
      pos += kBlockMetaBytes + 4ull * ((uint64_t)c.N + 1ull);
      c.b_off[4 * b + 2] = pos;
      pos += (c.b_N[b] * c.cb + 7ull) / 8ull;
      c.b_off[4 * b + 3] = pos;
      pos += (c.b_N[b] * c.b_q[b] + 7ull) / 8ull;
    }
    c.P = pos + kCrcBytes;
  }
  for (int b = tid; b < B; b += NT) {
    const double vmin = (double)__uint_as_float(c.b_min[b]), vmax = (double)__uint_as_float(c.b_max[b]);
    const bool degen = c.b_N[b] == 0 || c.b_min[b] == c.b_max[b];
    c.b_o64[b] = degen ? 1.0 : __ddiv_rn(__dsub_rn(vmax, vmin), (double)((1u << c.b_q[b]) - 1u));
    c.b_inv[b] = __drcp_rn(c.b_o64[b]);
  }
  __syncthreads();
  const uint64_t P = c.P;
  if (P > c.out_cap) return g;
  // codes at q* replace the value bits in the kept list (values are no longer needed)
  const List L = c.L;
  const Perm M = c.M;
  for (int b = 0; b < B; ++b) {
    const double vmin = (double)__uint_as_float(c.b_min[b]);
    const double o64 = c.b_o64[b], inv = c.b_inv[b];
    const uint32_t lv = (1u << c.b_q[b]) - 1u;
    const bool degen = c.b_min[b] == c.b_max[b];
    const uint32_t rs = c.b_rs[b], n = c.b_n[b];
    for (uint32_t i = tid; i < n; i += NT) {
      const uint32_t li = M.get(rs + i);
      const uint32_t code = degen ? 0u : quant_code(L.bits(li) & 0x7FFFFFFFu, vmin, o64, inv, lv);
      L.set_bits(li, code);
    }
  }
  uint8_t* out = c.out;
  const uint64_t z0 = P * g.rank / g.size, z1 = P * (g.rank + 1) / g.size;
  uint64_t za = (z0 + 15) & ~15ull, zb = z1 & ~15ull;
  if (za > zb) { za = z1; zb = z1; }
  for (uint64_t i = z0 + tid; i < za && i < z1; i += NT) out[i] = 0;
  for (uint64_t i = zb + tid; i < z1; i += NT) if (i >= za) out[i] = 0;
  uint4* o4 = reinterpret_cast<uint4*>(out);
  for (uint64_t i = za / 16 + tid; i < zb / 16; i += NT) o4[i] = make_uint4(0, 0, 0, 0);
  g.sync();  // CTA barrier / cluster barrier (release-acquire) orders the payload writes
  return g;
}

// ---- Phase I: header/meta, row_ptr, MSB-first word packing of cols and codes
template <int NT>
__device__ __noinline__ Grp phase_write(Ctx& c, Grp g, Shared& sh) {
  const int tid = threadIdx.x;
  const int B = c.B;
  const uint32_t N = c.N, K = c.K, cb = c.cb;
  uint8_t* out = c.out;
  if (g.rank == 0) {
    if (tid == 0) {
      uint8_t h[32];
      h[0] = 'S'; h[1] = 'I'; h[2] = 'F'; h[3] = '1';
      h[4] = 1; h[5] = 0;
      for (int k = 0; k < 4; ++k) { h[6 + k] = (uint8_t)(N >> (8 * k)); h[10 + k] = (uint8_t)(K >> (8 * k)); }
      const uint32_t s32 = __float_as_uint(__double2float_rn(c.s));
      const uint32_t l32 = __float_as_uint(__double2float_rn(c.lam));
      const uint32_t d32 = __float_as_uint(__double2float_rn(c.delta));
      for (int k = 0; k < 4; ++k) {
        h[14 + k] = (uint8_t)(s32 >> (8 * k));
        h[18 + k] = (uint8_t)(l32 >> (8 * k));
        h[23 + k] = (uint8_t)(d32 >> (8 * k));
      }
      h[22] = (uint8_t)c.q_bit;
      h[27] = (uint8_t)c.mode;
      h[28] = (uint8_t)c.meff[0]; h[29] = (uint8_t)(c.meff[0] >> 8);
      h[30] = (uint8_t)c.meff[1]; h[31] = (uint8_t)(c.meff[1] >> 8);
      for (int k = 0; k < 32; ++k) out[k] = h[k];
    }
    if (c.mode == SIF_MODE_FIXED)
      for (int b = tid; b < B; b += NT) out[kHeaderBytes + b] = (uint8_t)c.b_q[b];
    for (int b = tid; b < B; b += NT) {
      const uint64_t o = c.b_off[4 * b];
      out[o] = (uint8_t)c.b_q[b];
      st_u32_le_bytes(out, o + 1, __float_as_uint(c.b_N[b] == 0 ? 1.0f : __double2float_rn(c.b_o64[b])));
      st_u32_le_bytes(out, o + 5, c.b_N[b] == 0 ? 0u : c.b_min[b]);
      st_u32_le_bytes(out, o + 9, (uint32_t)c.b_N[b]);
    }
  }
  phase_mark(c, g, 12);
  const List L = c.L;
  const Perm M = c.M;
  const FastDiv fk = c.fk;
  // row_ptr (msplit.py:97-100): rows whose start r*K lies in [s0, s1); entry = number of
  // the block's members (group-wide) with flat index < r*K, by binary search
  {
    const uint32_t rfirst = (uint32_t)((c.s0 + K - 1) / K);
    const uint64_t rl = (c.s1 + K - 1) / K;  // exclusive
    const uint32_t rend = (uint32_t)(rl > N ? N : rl);
    const uint32_t nr = rend > rfirst ? rend - rfirst : 0;
    const uint32_t tot = nr * (uint32_t)B;
    for (uint32_t w = tid; w < tot; w += NT) {
      const int b = (int)(w / nr);
      const uint32_t r = rfirst + (w - (uint32_t)b * nr);
      const uint32_t bound = r * K;
      const uint32_t rs = c.b_rs[b];
      uint32_t lo = 0, hi = c.b_n[b];
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (L.idx(M.get(rs + mid)) < bound) lo = mid + 1; else hi = mid;
      }
      st_u32_le_bytes(out, c.b_off[4 * b + 1] + 4ull * r, (uint32_t)c.b_pre[b] + lo);
    }
    if (g.rank == g.size - 1)
      for (int b = tid; b < B; b += NT) st_u32_le_bytes(out, c.b_off[4 * b + 1] + 4ull * N, (uint32_t)c.b_N[b]);
  }
  phase_mark(c, g, 13);
  // cols / codes (bitstream.py:12-30): each job packs 8 consecutive fields of one
  // (block, section) MSB-first into a 64-bit window and emits payload-aligned 32-bit
  // words; words shared with a neighbouring job/section are merged with atomicOr.
  {
    uint32_t* out32 = reinterpret_cast<uint32_t*>(out);
    constexpr uint32_t FPJ = 8;
    uint32_t* jstart = reinterpret_cast<uint32_t*>(sh.pre);  // job prefix per block batch (<= 63 blocks)
    for (int bb0 = 0; bb0 < B; bb0 += 63) {
    const int Bj = B - bb0 < 63 ? B - bb0 : 63;
    __syncthreads();
    if (tid == 0) {
      uint32_t acc = 0;
      for (int k = 0; k < Bj; ++k) { jstart[k] = acc; acc += 2 * ((c.b_n[bb0 + k] + FPJ - 1) / FPJ); }
      jstart[Bj] = acc;
    }
    __syncthreads();
    const uint32_t njobs = jstart[Bj];
    for (uint32_t job = tid; job < njobs; job += NT) {
      int bk = 0;
      while (bk + 1 < Bj && jstart[bk + 1] <= job) ++bk;
      const uint32_t jj = job - jstart[bk];
      const int b = bb0 + bk;
      const uint32_t nloc = c.b_n[b];
      const uint32_t ng = (nloc + FPJ - 1) / FPJ;
      const int sec = jj < ng ? 0 : 1;
      const uint32_t gi = sec ? jj - ng : jj;
      const uint64_t pre = c.b_pre[b];
      const uint32_t rs = c.b_rs[b];
      const uint32_t w = sec == 0 ? cb : c.b_q[b];
      const uint32_t f0 = gi * FPJ, f1 = f0 + FPJ < nloc ? f0 + FPJ : nloc;
      const uint64_t bit = 8ull * c.b_off[4 * b + 2 + sec] + (pre + f0) * (uint64_t)w;
      const uint64_t lo_bit = bit, hi_bit = bit + (uint64_t)(f1 - f0) * w;
      uint64_t wbase = bit & ~31ull;
      uint64_t acc = 0;
      uint32_t nacc = (uint32_t)(bit - wbase);
      uint32_t vv[FPJ];
#pragma unroll
      for (uint32_t k = 0; k < FPJ; ++k) {
        vv[k] = 0;
        if (f0 + k < f1) {
          const uint32_t li = M.get(rs + f0 + k);
          vv[k] = sec == 0 ? fk.mod(L.idx(li)) : L.bits(li);
        }
      }
#pragma unroll
      for (uint32_t k = 0; k < FPJ; ++k) {
        if (f0 + k < f1) {
          acc |= (uint64_t)vv[k] << (64u - nacc - w);
          nacc += w;
          if (nacc >= 32) {
            const uint32_t word = (uint32_t)(acc >> 32);
            const uint64_t wa = wbase >> 5;
            if (wbase >= lo_bit) out32[wa] = bswap32(word);
            else if (word) atomicOr(out32 + wa, bswap32(word));
            acc <<= 32;
            nacc -= 32;
            wbase += 32;
          }
        }
      }
      if (nacc) {
        const uint32_t word = (uint32_t)(acc >> 32);
        const uint64_t wa = wbase >> 5;
        if (wbase >= lo_bit && wbase + 32 <= hi_bit) out32[wa] = bswap32(word);
        else if (word) atomicOr(out32 + wa, bswap32(word));
      }
    }
    }
  }
  g.sync();  // CTA barrier / cluster barrier (release-acquire) orders the payload writes
  return g;
}

// ---- Phase J: CRC-32 over bytes [4, P-4) (codec.py:316); rounds interleaved over the group
template <int NT>
__device__ __noinline__ void phase_crc(Ctx& c, Grp g, Shared& sh, uint64_t* out_len, int32_t* status) {
  const uint64_t P = c.P;
  uint32_t part;
  if (c.L.cap * 12u >= (uint32_t)(NT * 64))
    part = crc_cta_staged<NT>(c.out, 4, P - 4, c.t4, sh.red, c.L.sb, g.rank, g.size);
  else
    part = g.rank == 0 ? crc_cta_raw<NT>(c.out, 4, P - 4, c.t4, sh.red) : 0u;
  uint32_t total = part;
  if (g.size > 1) {
    uint64_t* slot = g.slot();
    if (threadIdx.x == 0) slot[0] = part;
    g.sync();
    if (g.rank == 0 && threadIdx.x == 0) {
      cg::cluster_group cl = cg::this_cluster();
      total = 0;
      for (uint32_t r = 0; r < g.size; ++r) total ^= (uint32_t)*cl.map_shared_rank(slot, r);
    }
    g.parity ^= 1;
  }
  if (g.rank == 0 && threadIdx.x == 0) {
    st_u32_le_bytes(c.out, P - 4, crc_finish(total, P - 8));
    if (c.prof) c.prof[(uint64_t)c.ifi * 32 + 15] = gtimer();
    out_len[c.ifi] = P;
    status[c.ifi] = SIF_OK;
  }
}

// ---------------------------------------------------------------------------------------
template <int DT, int NT>
__device__ __forceinline__ void encode_one(const EncArgs& a, Ctx& c, Grp g, Shared& sh) {
  phase_mark(c, g, 0);
  g = phase_sample<DT, NT>(c, g, sh);
  phase_mark(c, g, 1);
  g = phase_stream<DT, NT>(c, g, sh);
  if (c.nonfinite) {
    if (g.rank == 0 && threadIdx.x == 0) { a.status[c.ifi] = SIF_ERR_NONFINITE; if (!a.atkf_only) a.out_len[c.ifi] = 0; }
    return;
  }
  phase_mark(c, g, 2);
  g = phase_select<NT>(c, g, sh);
  phase_mark(c, g, 4);
  g = phase_kept<NT>(c, g, sh);
  if (a.atkf_only) {
    int64_t* out = a.kept_out + a.kept_off[c.ifi] + c.kept_pre;
    for (uint32_t i = threadIdx.x; i < c.nkept; i += NT) out[i] = (int64_t)c.L.idx(i);
    if (g.rank == 0 && threadIdx.x == 0) {
      a.tau3[3 * c.ifi + 0] = c.tau;
      a.tau3[3 * c.ifi + 1] = c.tau_p;
      a.tau3[3 * c.ifi + 2] = c.tau_m;
      a.status[c.ifi] = SIF_OK;
    }
    return;
  }
  phase_mark(c, g, 6);
  g = phase_cuts<NT>(c, g, sh);
  phase_mark(c, g, 7);
  g = phase_members<NT>(c, g, sh, a.scratch_words * 4);
  phase_mark(c, g, 8);
  g = phase_minmax<NT>(c, g, sh);
  phase_mark(c, g, 9);
  g = phase_abq<NT>(c, g, sh);
  phase_mark(c, g, 10);
  g = phase_layout<NT>(c, g, sh);
  if (c.P > c.out_cap) {
    if (g.rank == 0 && threadIdx.x == 0) { a.status[c.ifi] = SIF_ERR_CAPACITY; a.out_len[c.ifi] = c.P; }
    return;
  }
  phase_mark(c, g, 11);
  g = phase_write<NT>(c, g, sh);
  phase_mark(c, g, 14);
  phase_crc<NT>(c, g, sh, a.out_len, a.status);
}

template <int NT>
__global__ void __launch_bounds__(NT, (NT == 512 ? 1 : 2)) sif_encode_kernel(EncArgs a) {
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ Shared sh;
  __shared__ Ctx c;
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
  if (threadIdx.x == 0) {
    const sif_enc_desc d = a.descs[ifi];
    c.x = d.x; c.out = d.out; c.out_cap = d.out_cap; c.seed = d.seed;
    c.N = d.rows; c.K = d.cols; c.dtype = d.dtype; c.cb = col_bits(d.cols);
    c.T = (uint64_t)d.rows * d.cols;
    c.s0 = c.T * g.rank / g.size;
    c.s1 = c.T * (g.rank + 1) / g.size;
    c.kk = keep_count(a.s, c.T);
    c.fk.init(d.cols);
    c.s = a.s; c.lam = a.lam; c.delta = a.delta;
    c.m_plus = a.m_plus; c.m_minus = a.m_minus; c.q_bit = a.q_bit; c.mode = a.mode;
    c.atkf_only = a.atkf_only; c.maxb = a.maxb; c.ifi = ifi;
    c.fixed_q = a.fixed_q;
    c.prof = a.prof;
    const int maxb = a.maxb, NW = NT / 32;
    c.t4 = reinterpret_cast<uint32_t*>(dsm);
    c.scratch = c.t4 + 1024;
    uint8_t* p = reinterpret_cast<uint8_t*>(c.scratch + a.scratch_words);
    c.b_sum = reinterpret_cast<uint64_t*>(p); p += 8ull * maxb;
    c.b_pre = reinterpret_cast<uint64_t*>(p); p += 8ull * maxb;
    c.b_N = reinterpret_cast<uint64_t*>(p); p += 8ull * maxb;
    c.b_off = reinterpret_cast<uint64_t*>(p); p += 8ull * 4 * maxb;
    c.b_o64 = reinterpret_cast<double*>(p); p += 8ull * maxb;
    c.b_inv = reinterpret_cast<double*>(p); p += 8ull * maxb;
    c.b_n = reinterpret_cast<uint32_t*>(p); p += 4ull * maxb;
    c.b_rs = reinterpret_cast<uint32_t*>(p); p += 4ull * maxb;
    c.b_min = reinterpret_cast<uint32_t*>(p); p += 4ull * maxb;
    c.b_max = reinterpret_cast<uint32_t*>(p); p += 4ull * maxb;
    c.b_q = reinterpret_cast<uint32_t*>(p); p += 4ull * maxb;
    c.b_act = reinterpret_cast<uint32_t*>(p); p += 4ull * maxb;
    c.cut_key = reinterpret_cast<uint32_t*>(p); p += 4ull * maxb;
    c.cut_idx = reinterpret_cast<uint32_t*>(p); p += 4ull * maxb;
    c.wcnt = reinterpret_cast<uint32_t*>(p); p += 4ull * NW * maxb;
    c.woff = reinterpret_cast<uint32_t*>(p); p += 4ull * NW * maxb;
    p = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
    const uint32_t cap = (uint32_t)a.cap;
    uint8_t* spill = a.spill + a.spill_stride * ((uint64_t)ifi * g.size + g.rank);
    const uint64_t slice = c.s1 - c.s0;
    const uint64_t spill_n = slice > cap ? slice - cap : 0;
    c.L.sb = reinterpret_cast<uint32_t*>(p);
    c.L.si = c.L.sb + cap;
    c.L.gb = reinterpret_cast<uint32_t*>(spill);
    c.L.gi = c.L.gb + spill_n;
    c.L.cap = cap;
    c.M.s = c.L.si + cap;
    c.M.g = c.L.gi + spill_n;
    c.M.cap = cap;
  }
  for (int i = threadIdx.x; i < 1024; i += NT) reinterpret_cast<uint32_t*>(dsm)[i] = (&kCrcTab4[0][0])[i];
  __syncthreads();
  if (c.dtype == SIF_DTYPE_BF16) encode_one<SIF_DTYPE_BF16, NT>(a, c, g, sh);
  else encode_one<SIF_DTYPE_F32, NT>(a, c, g, sh);
  if (g.size > 1) cg::this_cluster().sync();  // keep DSMEM alive until all peers are done
}

template __global__ void sif_encode_kernel<256>(EncArgs);
template __global__ void sif_encode_kernel<512>(EncArgs);

}  // namespace sif
