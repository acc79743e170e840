// sif_lib.cu -- C ABI (include/sif.h) of the B200 SLICER IF codec: planning, workspace
// layout, uploads and kernel launches.  One translation unit: the kernels are included.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <vector>

#include "sif.h"
#include "sif_decode.cu"
#include "sif_token.cu"
#include "sif_synth.cu"

namespace {


inline uint64_t up(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

int check_cuda(cudaError_t e) { return e == cudaSuccess ? SIF_OK : SIF_ERR_CUDA; }

// ---- optional per-kernel timing (diagnostics; sif_profile_enable)
enum { KP_PREP, KP_STREAM, KP_SELECT, KP_MEMBERS, KP_ABQ1, KP_ABQ2, KP_LAYOUT, KP_PACK, KP_CRC, KP_PARSE, KP_DCRC,
       KP_SCATTER, KP_DFINAL, KP_SELECT_TINY, KP_GATHER1, KP_SELECT1, KP_GATHER2, KP_SELECT2, KP_FUSED, KP_TOKEN, KP_DSMALL, KP_N };
const char* kKpNames[KP_N] = {"enc_prep", "enc_stream", "enc_select<0>", "enc_members", "enc_abq<1>", "enc_abq<0>",
                              "enc_layout", "enc_pack", "enc_crc", "sif_parse_kernel", "sif_dcrc_kernel",
                              "sif_scatter_kernel", "sif_dfinal_kernel", "enc_select_tiny", "enc_gather<1>",
                              "enc_select<1>", "enc_gather<2>", "enc_select<2>", "enc_post", "enc_token",
                              "sif_dec_small"};
struct ProfRec { int k; cudaEvent_t a, b; };
std::atomic<bool> g_prof{false};
std::mutex g_prof_mu;  // guards g_recs (launches may come from several host threads)
std::vector<ProfRec> g_recs;
struct ProfScope {
  int k;
  cudaStream_t s;
  cudaEvent_t a = nullptr, b = nullptr;
  ProfScope(int kk, cudaStream_t ss) : k(kk), s(ss) {
    if (!g_prof.load(std::memory_order_relaxed)) return;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
  }
  ~ProfScope() {
    if (!a) return;
    cudaEventRecord(b, s);
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_recs.push_back({k, a, b});
  }
};

// Host GF(2) arithmetic for the CRC-32 segment shift table (same as sif_common.cuh).
uint32_t h_crc_mult(uint32_t a, uint32_t b) {
  uint32_t p = 0;
  for (int i = 31; i >= 0; --i) {
    p ^= b & (0u - ((a >> i) & 1u));
    b = (b >> 1) ^ (0xEDB88320u & (0u - (b & 1u)));
  }
  return p;
}
uint32_t h_x8n(uint64_t nbytes) {  // x^(8 n) mod P, reflected
  uint32_t x2n[64];
  x2n[0] = 1u << 30;  // x^1
  for (int k = 1; k < 64; ++k) x2n[k] = h_crc_mult(x2n[k - 1], x2n[k - 1]);
  uint32_t p = 1u << 31;  // x^0
  int k = 3;
  while (nbytes) {
    if (nbytes & 1ull) p = h_crc_mult(x2n[k & 63], p);
    nbytes >>= 1;
    ++k;
  }
  return p;
}

// Fraction of the resident CTA slots a persistent kernel takes (SIF_GRID_FRAC, default 1):
// below 1 leaves room for kernels of other in-flight batches on other streams.
double grid_frac() {
  static const double f = [] {
    const char* e = getenv("SIF_GRID_FRAC");
    const double v = e && *e ? atof(e) : 1.0;
    return (v > 0.0 && v <= 1.0) ? v : 1.0;
  }();
  return f;
}

template <class K>
int resident_grid(K kfn, int threads, int smem, uint64_t work, int sms) {
  int per = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kfn, threads, smem) != cudaSuccess || per < 1) per = 1;
  const uint64_t slots = std::max<uint64_t>(1, (uint64_t)(per * sms * grid_frac()));
  return (int)std::max<uint64_t>(1, std::min<uint64_t>(work, slots));
}

// Candidates above which an IF uses the multi-kernel select (all-SM gathers); env
// SIF_BIG_NCAND overrides it (tuning experiments).
static uint32_t big_ncand() {
  static const uint32_t v = [] {
    const char* e = getenv("SIF_BIG_NCAND");
    return e && *e ? (uint32_t)strtoul(e, nullptr, 0) : 131072u;
  }();
  return v;
}
constexpr int kSmemStream = (2 * sif::CH + 2 * sif::ND) * 4;
constexpr int kSmemSelect = (2 * sif::ND + 2 * sif::HB + sif::GCAP * 4 + 2 * sif::GSM) * 4;
inline int smem_abq(int maxb) { return (sif::CNT / 32) * maxb * (int)(sizeof(sif::AbqPar) + 16 * 8); }
inline int smem_pack(int maxb) { return (sif::CNT / 32) * maxb * (int)sizeof(sif::PackPar); }
inline uint32_t crc_segments(uint64_t cap) { return (uint32_t)std::max<uint64_t>(1, (cap + sif::CRC_PIECE - 1) / sif::CRC_PIECE); }
constexpr int kSmemScatterMax = (sif::DNT / 32) * 2 * ((4096 + 31) / 32) * 4;

// Per-device state: everything that depends on the device a call runs on (the CRC piece
// shift table in that device's __constant__/__device__ memory, kernel attributes, SM
// count, resident grid sizes).  Initialised once per device on first use; a process may
// drive several GPUs (one host thread per GPU, or one thread switching devices).
struct DevState {
  std::once_flag once;
  int status = SIF_OK;
  int sms = 148;
  int g_stream = 1, g_members = 1, g_gather = 1, g_crc = 1, g_dcrc = 1, g_scatter = 1;
  int post_smem = 0;       // enc_post: dynamic shared memory (all that is left next to its static part)
  uint32_t post_lcap = 0;  // enc_post: candidates held in shared memory
  std::mutex mu;  // guards the per-maxb grid cache
  int g_abq[sif::MAXB + 1] = {0};
  int g_pack[sif::MAXB + 1] = {0};
};
constexpr int kMaxDevices = 64;
DevState g_dev[kMaxDevices];

int dev_init(DevState& ds, int dev) {
  if (cudaDeviceGetAttribute(&ds.sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || ds.sms <= 0) ds.sms = 148;
  std::vector<uint32_t> t(sif::CRC_PIECES_MAX);
  const uint32_t step = h_x8n(sif::CRC_PIECE);
  t[0] = 1u << 31;
  for (int j = 1; j < sif::CRC_PIECES_MAX; ++j) t[j] = h_crc_mult(step, t[j - 1]);
  if (cudaMemcpyToSymbol(sif::kPieceShift, t.data(), 4ull * sif::CRC_PIECES_MAX) != cudaSuccess) return SIF_ERR_CUDA;
  if (check_cuda(cudaFuncSetAttribute(sif::enc_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemStream)) ||
      check_cuda(cudaFuncSetAttribute(sif::enc_select<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemSelect)) ||
      check_cuda(cudaFuncSetAttribute(sif::enc_select<0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemSelect)) ||
      check_cuda(cudaFuncSetAttribute(sif::enc_select<0, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemSelect)) ||
      check_cuda(cudaFuncSetAttribute(sif::enc_select<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemSelect)) ||
      check_cuda(cudaFuncSetAttribute(sif::enc_select<1, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemSelect)) ||
      check_cuda(cudaFuncSetAttribute(sif::enc_select<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemSelect)) ||

      check_cuda(cudaFuncSetAttribute(sif::enc_abq<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_abq(32))) ||
      check_cuda(cudaFuncSetAttribute(sif::enc_abq<0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_abq(32))) ||
      check_cuda(cudaFuncSetAttribute(sif::enc_pack<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_pack(32))) ||
      check_cuda(cudaFuncSetAttribute(sif::enc_abq<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_abq(sif::MAXB))) ||
      check_cuda(cudaFuncSetAttribute(sif::enc_abq<0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_abq(sif::MAXB))) ||
      check_cuda(cudaFuncSetAttribute(sif::enc_pack<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_pack(sif::MAXB))) ||
      check_cuda(cudaFuncSetAttribute(sif::sif_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kSmemScatterMax)))
    return SIF_ERR_CUDA;
  {
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, sif::enc_post) != cudaSuccess) return SIF_ERR_CUDA;
    int optin = 0;
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) return SIF_ERR_CUDA;
    ds.post_smem = optin - (int)fa.sharedSizeBytes;
    if (ds.post_smem < sif::kSmemSelectBytes + 8 * 1024) return SIF_ERR_CUDA;
    ds.post_lcap = (uint32_t)((ds.post_smem - sif::kSmemSelectBytes) / 8);
    if (check_cuda(cudaFuncSetAttribute(sif::enc_post, cudaFuncAttributeMaxDynamicSharedMemorySize, ds.post_smem)))
      return SIF_ERR_CUDA;
  }
  const uint64_t big = 1ull << 30;
  ds.g_gather = resident_grid(sif::enc_gather<1>, sif::CNT, 0, big, ds.sms);
  ds.g_crc = resident_grid(sif::enc_crc, sif::CNT, 0, big, ds.sms);
  ds.g_stream = resident_grid(sif::enc_stream, sif::CNT, kSmemStream, big, ds.sms);
  ds.g_members = resident_grid(sif::enc_members, sif::CNT, 0, big, ds.sms);
  ds.g_dcrc = resident_grid(sif::sif_dcrc_kernel, sif::DNT, 0, big, ds.sms);
  return SIF_OK;
}

// State of the calling thread's current device (initialised on first use), or nullptr.
DevState* dev_state() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return nullptr;
  DevState& ds = g_dev[dev];
  std::call_once(ds.once, [&] { ds.status = dev_init(ds, dev); });
  return ds.status == SIF_OK ? &ds : nullptr;
}

// Workspace sections of an encode plan (all offsets 256-byte aligned).
struct EncWs {
  uint64_t info, st, ch_if, ch_e0, u_off, u_cnt, bcnt, bpre, brs, blast, bprev, hist, fixedq, keptoff, segbase, biglist,
      fused, tokens, lists;
};

EncWs enc_ws(uint64_t n, uint64_t nch, uint64_t maxb, uint64_t nhist, uint64_t nq) {
  EncWs w;
  uint64_t off = 0;
  auto take = [&](uint64_t bytes) { const uint64_t o = off; off += up(std::max<uint64_t>(bytes, 1), 256); return o; };
  w.info = take(sizeof(sif::IfInfo) * n);
  w.st = take(sizeof(sif::IfSt) * n);
  w.ch_if = take(4 * nch);
  w.ch_e0 = take(4 * nch);
  w.u_off = take(4 * nch * sif::UNITS);
  w.u_cnt = take(4 * nch * sif::UNITS);
  w.bcnt = take(4 * nch * maxb);
  w.bpre = take(4 * nch * maxb);
  w.brs = take(4 * nch * maxb);
  w.blast = take(4 * nch * maxb);
  w.bprev = take(4 * nch * maxb);
  w.hist = take(4ull * 2 * sif::ND * nhist);
  w.fixedq = take(nq);
  w.keptoff = take(8 * n);
  w.segbase = take(4 * (n + 1));
  w.biglist = take(4 * (n + 1));
  w.fused = take(4 * (n + 1));
  w.tokens = take(4 * (n + 1));
  w.lists = off;
  return w;
}

}  // namespace

extern "C" {

int sif_version(void) { return 1; }

int sif_profile_enable(int on) {
  g_prof.store(on != 0);
  return SIF_OK;
}

int sif_profile_enabled(void) { return g_prof.load() ? 1 : 0; }

int sif_profile_read(double* ms, int32_t* count, int maxk) {
  if (!ms || !count || maxk < 0) return SIF_ERR_INVALID_ARG;
  for (int k = 0; k < maxk; ++k) { ms[k] = 0.0; count[k] = 0; }
  int st = SIF_OK;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (const ProfRec& r : g_recs) {
    float t = 0.f;
    if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess) st = SIF_ERR_CUDA;
    if (r.k < maxk) { ms[r.k] += t; count[r.k] += 1; }
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_recs.clear();
  return st ? -st : KP_N;
}

const char* sif_profile_kernel_name(int k) { return k >= 0 && k < KP_N ? kKpNames[k] : ""; }

uint64_t sif_keep_count(double s, uint64_t t) { return sif::keep_count(s, t); }

uint32_t sif_col_bits(uint32_t k) { return sif::col_bits(k); }

const char* sif_status_string(int st) {
  switch (st) {
    case SIF_OK: return "ok";
    case SIF_ERR_CONFIG: return "ConfigError";
    case SIF_ERR_NONFINITE: return "NonFiniteError";
    case SIF_ERR_SHAPE: return "ShapeError";
    case SIF_ERR_STREAM_FORMAT: return "StreamFormatError";
    case SIF_ERR_CORRUPT_STREAM: return "CorruptStreamError";
    case SIF_ERR_CAPACITY: return "CapacityError";
    case SIF_ERR_CUDA: return "CudaError";
    case SIF_ERR_INVALID_ARG: return "InvalidArgument";
    default: return "unknown";
  }
}

// codec.py:72-92
int sif_validate_cfg(const sif_codec_cfg* c) {
  if (!c) return SIF_ERR_INVALID_ARG;
  if (!(c->s >= 0.0 && c->s <= 1.0)) return SIF_ERR_CONFIG;
  if (!(c->lam >= 0.0 && c->lam < 1.0)) return SIF_ERR_CONFIG;
  if (c->m_plus < 1 || c->m_minus < 1) return SIF_ERR_CONFIG;
  if (c->q_bit < 1 || c->q_bit > 16) return SIF_ERR_CONFIG;
  if (!(c->delta >= 0.0)) return SIF_ERR_CONFIG;
  if (c->mode != SIF_MODE_ABQ && c->mode != SIF_MODE_FIXED) return SIF_ERR_CONFIG;
  if (c->mode == SIF_MODE_FIXED) {
    if (!c->fixed_q) return SIF_ERR_CONFIG;
    for (int i = 0; i < c->m_plus + c->m_minus; ++i)
      if (c->fixed_q[i] < 1 || c->fixed_q[i] > 16) return SIF_ERR_CONFIG;
  }
  if (c->m_plus > 65535 || c->m_minus > 65535) return SIF_ERR_CONFIG;
  return SIF_OK;
}

// Sound capacity bound (planner.py:33-64 charges q_bit only, which under-counts fixed-Q
// blocks with q > q_bit; here every block is charged max(q_bit, max fixed q)).
uint64_t sif_max_payload_bytes(uint32_t rows, uint32_t cols, const sif_codec_cfg* c) {
  if (sif_validate_cfg(c) != SIF_OK) return 0;
  const uint64_t T = (uint64_t)rows * cols;
  const uint64_t k = sif::keep_count(c->s, T);
  uint32_t qmax = (uint32_t)c->q_bit;
  if (c->mode == SIF_MODE_FIXED)
    for (int i = 0; i < c->m_plus + c->m_minus; ++i) qmax = std::max<uint32_t>(qmax, c->fixed_q[i]);
  const uint64_t kk = std::max<uint64_t>(1, k);
  const uint64_t B = std::min<uint64_t>(c->m_plus, kk) + std::min<uint64_t>(c->m_minus, kk);
  uint64_t bytes = 36 + (c->mode == SIF_MODE_FIXED ? B : 0);
  bytes += B * (13 + 4ull * ((uint64_t)rows + 1) + 2);
  bytes += (k * (sif::col_bits(cols) + qmax) + 7) / 8;
  return up(bytes, 16);
}

// ------------------------------------------------------------------ encode
// IFs of [tmin, tmax] elements (env SIF_FUSED_MIN / SIF_FUSED_MAX, or sif_set_fused_range;
// default: none) take the per-IF back end after the stream pass (one CTA per IF from the
// candidate list to the .sif stream, sif_post.cu); the others the chunk kernels.  Only
// multi-chunk IFs qualify.  Read when a plan is made.  Measured on C2 (256 x 1024x196): the
// per-IF back end is correct but slower than the chunk kernels in the pipelined steady
// state (one 1024-thread CTA per SM holds ~210 KB of shared memory, so other slots' kernels
// cannot co-reside, and the passes execute more instructions), hence off by default.
static std::atomic<uint64_t> g_fmin{0}, g_fmax{0};
static std::once_flag g_frange_once;
static void fused_range(uint64_t& tmin, uint64_t& tmax) {
  std::call_once(g_frange_once, [] {
    const char* e0 = getenv("SIF_FUSED_MIN");
    const char* e1 = getenv("SIF_FUSED_MAX");
    g_fmin = e0 && *e0 ? strtoull(e0, nullptr, 0) : 1ull;
    g_fmax = e1 && *e1 ? strtoull(e1, nullptr, 0) : 0ull;
  });
  tmin = g_fmin.load();
  tmax = g_fmax.load();
}
static bool is_fused(uint64_t T, int atkf) {
  uint64_t tmin, tmax;
  fused_range(tmin, tmax);
  return !atkf && T > (uint64_t)sif::CH && T < (1ull << 25) && T >= tmin && T <= tmax;
}

// Token path: IFs of <= 4096 elements with lambda = 0, k >= 1 and at most 8 blocks are
// encoded start to finish by enc_token (one CTA each); SIF_TOKEN=0 turns it off.
static bool is_token(uint64_t T, int atkf, const sif_codec_cfg* c) {
  static const bool on = [] { const char* e = getenv("SIF_TOKEN"); return !(e && *e == '0'); }();
  if (!on || atkf || T > (uint64_t)sif::KT || c->lam != 0.0) return false;
  const uint64_t k = sif::keep_count(c->s, T);
  if (k < 1) return false;
  return std::min<uint64_t>(c->m_plus, k) + std::min<uint64_t>(c->m_minus, k) <= (uint64_t)sif::KB;
}

static int enc_plan_impl(const sif_enc_desc* d, int n, const sif_codec_cfg* c, int atkf, sif_plan* p) {
  if (!d || !p || n < 0) return SIF_ERR_INVALID_ARG;
  int st = sif_validate_cfg(c);
  if (st) return st;
  memset(p, 0, sizeof(*p));
  uint64_t kmax = 0, nch = 0, nhist = 0, lists = 0, nseg = 0;
  bool tiny = false;  // some IF may take the warp-per-IF select (enc_select_tiny)
  bool all_small = n > 0;  // every IF fits one chunk: narrow enc_prep
  int nfused = 0, ntoken = 0;
  for (int i = 0; i < n; ++i) {
    if (d[i].rows < 1 || d[i].cols < 1) return SIF_ERR_SHAPE;  // tensor.py:27-28
    const uint64_t T = (uint64_t)d[i].rows * d[i].cols;
    if (T >= (1ull << 31)) return SIF_ERR_INVALID_ARG;
    if (d[i].dtype != SIF_DTYPE_F32 && d[i].dtype != SIF_DTYPE_BF16) return SIF_ERR_INVALID_ARG;
    if (!d[i].x || (reinterpret_cast<uintptr_t>(d[i].x) & 15)) return SIF_ERR_INVALID_ARG;
    if (!atkf && (!d[i].out || (reinterpret_cast<uintptr_t>(d[i].out) & 15))) return SIF_ERR_INVALID_ARG;
    if (sif_max_payload_bytes(d[i].rows, d[i].cols, c) >= (1ull << 29)) return SIF_ERR_INVALID_ARG;  // u32 bit offsets
    if (crc_segments(d[i].out_cap) > (uint64_t)sif::CRC_PIECES_MAX) return SIF_ERR_INVALID_ARG;
    if (is_token(T, atkf, c)) {  // enc_token does it all
      ++ntoken;
      lists += up(16 * T, 256);
      continue;
    }
    const uint64_t ch = (T + sif::CH - 1) / sif::CH;
    nch += ch;
    if (ch > 1) ++nhist;
    if (ch > 1) all_small = false;
    if (is_fused(T, atkf)) {  // stream pass as the pipeline, then enc_post
      ++nfused;
      lists += up(24 * T, 256);
      continue;
    }
    lists += up(16 * T, 256);
    kmax = std::max(kmax, sif::keep_count(c->s, T));
    if (ch == 1 && !atkf && c->lam == 0.0 && sif::keep_count(c->s, T) > 0) tiny = true;
    nseg += crc_segments(d[i].out_cap);
  }
  if (nch >= (1ull << 31) || nseg >= (1ull << 31)) return SIF_ERR_INVALID_ARG;
  uint64_t kall = kmax;  // the block bound covers the fused IFs too
  for (int i = 0; i < n; ++i) kall = std::max(kall, sif::keep_count(c->s, (uint64_t)d[i].rows * d[i].cols));
  const uint64_t kk = std::max<uint64_t>(1, kall);
  const int maxb = (int)(std::min<uint64_t>(c->m_plus, kk) + std::min<uint64_t>(c->m_minus, kk));
  static_assert(sif::MAXB == SIF_MAX_BLOCKS, "sif.h SIF_MAX_BLOCKS");
  if (maxb > sif::MAXB) return SIF_ERR_CONFIG;  // more blocks than the encoder supports
  const EncWs w = enc_ws(n, nch, maxb, nhist, (uint64_t)c->m_plus + c->m_minus);
  p->n = n;
  p->cluster = (int32_t)nseg;  // encode plans: CRC segments (grid of enc_crc)
  p->threads = sif::CNT;
  p->smem_bytes = kSmemSelect;
  p->cap_smem = (int32_t)nhist;
  p->max_blocks = maxb;
  p->tiles = (int32_t)nch;
  // bit 0: ATKF-only, bit 1: multi-kernel select, bit 2: warp-per-IF select for small IFs,
  // bit 3: every IF fits one chunk (narrow enc_prep)
  p->flags = atkf | (kmax * 2 > (uint64_t)big_ncand() ? 2 : 0) | (tiny ? 4 : 0) | (all_small ? 8 : 0);
  p->ws_desc_off = w.info;
  p->ws_aux_off = w.fixedq;
  p->ws_spill_off = w.lists;
  p->ws_bytes = w.lists + lists;
  p->n_fused = nfused;
  p->reserved = ntoken;  // encode plans: IFs on the token path
  if (ntoken == n) p->flags &= ~8;  // no pipeline IF: nothing to narrow
  return SIF_OK;
}

static std::atomic<uint64_t> g_routing_epoch{0};  // bumped by every routing setter

int sif_set_fused_range(uint64_t tmin, uint64_t tmax) {
  uint64_t a, b;
  fused_range(a, b);  // env defaults first, then the override
  g_fmin = tmin;
  g_fmax = tmax;
  g_routing_epoch.fetch_add(1);
  return SIF_OK;
}

uint64_t sif_routing_epoch(void) { return g_routing_epoch.load(); }

int sif_get_fused_range(uint64_t* tmin, uint64_t* tmax) {
  if (!tmin || !tmax) return SIF_ERR_INVALID_ARG;
  fused_range(*tmin, *tmax);
  return SIF_OK;
}

int sif_enc_plan(const sif_enc_desc* d, int n, const sif_codec_cfg* c, sif_plan* p) {
  return enc_plan_impl(d, n, c, 0, p);
}

int sif_enc_upload(const sif_plan* p, const sif_enc_desc* d, const sif_codec_cfg* c, void* ws, void* stream) {
  if (!p || !ws || !c || (p->n > 0 && !d)) return SIF_ERR_INVALID_ARG;
  if (!dev_state()) return SIF_ERR_CUDA;
  cudaStream_t s = (cudaStream_t)stream;
  uint8_t* wb = (uint8_t*)ws;
  const int n = p->n;
  const EncWs w = enc_ws(n, (uint64_t)p->tiles, p->max_blocks, (uint64_t)p->cap_smem, (uint64_t)c->m_plus + c->m_minus);
  std::vector<sif::IfInfo> info((size_t)std::max(n, 1));
  std::vector<uint32_t> ch_if((size_t)std::max(p->tiles, 1)), ch_e0((size_t)std::max(p->tiles, 1));
  std::vector<uint32_t> seg((size_t)n + 1, 0);
  std::vector<uint32_t> fused, tokens;
  uint64_t ch = 0, lists = w.lists;
  int32_t hs = 0;
  for (int i = 0; i < n; ++i) {
    sif::IfInfo& f = info[i];
    memset(&f, 0, sizeof(f));
    f.x = d[i].x;
    f.out = d[i].out;
    // bytes past the largest possible payload are never touched (zeroing in enc_members)
    f.cap = std::min<uint64_t>(d[i].out_cap, sif_max_payload_bytes(d[i].rows, d[i].cols, c));
    f.seed = d[i].seed;
    f.T = (uint64_t)d[i].rows * d[i].cols;
    f.kk = sif::keep_count(c->s, f.T);
    f.N = d[i].rows;
    f.K = d[i].cols;
    f.cb = sif::col_bits(d[i].cols);
    f.dtype = d[i].dtype;
    const uint64_t nc = is_token(f.T, p->flags & 1, c) ? 0 : (f.T + sif::CH - 1) / sif::CH;
    f.ch0 = (uint32_t)ch;
    f.nch = (uint32_t)nc;
    f.hslot = nc > 1 ? hs++ : -1;
    f.list_off = lists;
    f.gat_off = lists + 8 * f.T;
    f.path = sif::PATH_PIPE;
    if (is_token(f.T, p->flags & 1, c)) {
      f.path = sif::PATH_TOKEN;
      f.ch0 = 0;
      f.nch = 0;
      f.hslot = -1;
      lists += up(16 * f.T, 256);
      seg[i + 1] = seg[i];
      tokens.push_back((uint32_t)i);
      continue;
    }
    if (is_fused(f.T, p->flags & 1)) {  // no CRC pieces: enc_post finishes the stream
      f.path = sif::PATH_POST;
      f.sp_off = lists + 16 * f.T;
      lists += up(24 * f.T, 256);
      seg[i + 1] = seg[i];
      fused.push_back((uint32_t)i);
    } else {
      lists += up(16 * f.T, 256);
      seg[i + 1] = seg[i] + crc_segments(f.cap);
    }
    for (uint64_t k = 0; k < nc; ++k) {
      ch_if[ch + k] = (uint32_t)i;
      ch_e0[ch + k] = (uint32_t)(k * sif::CH);
    }
    ch += nc;
  }
  if (n > 0) {
    if (check_cuda(cudaMemcpyAsync(wb + w.info, info.data(), sizeof(sif::IfInfo) * n, cudaMemcpyHostToDevice, s)))
      return SIF_ERR_CUDA;
    if (check_cuda(cudaMemcpyAsync(wb + w.ch_if, ch_if.data(), 4ull * ch, cudaMemcpyHostToDevice, s)))
      return SIF_ERR_CUDA;
    if (check_cuda(cudaMemcpyAsync(wb + w.ch_e0, ch_e0.data(), 4ull * ch, cudaMemcpyHostToDevice, s)))
      return SIF_ERR_CUDA;
    if (check_cuda(cudaMemcpyAsync(wb + w.segbase, seg.data(), 4ull * (n + 1), cudaMemcpyHostToDevice, s)))
      return SIF_ERR_CUDA;
    if (!fused.empty() &&
        check_cuda(cudaMemcpyAsync(wb + w.fused, fused.data(), 4ull * fused.size(), cudaMemcpyHostToDevice, s)))
      return SIF_ERR_CUDA;
    if (!tokens.empty() &&
        check_cuda(cudaMemcpyAsync(wb + w.tokens, tokens.data(), 4ull * tokens.size(), cudaMemcpyHostToDevice, s)))
      return SIF_ERR_CUDA;
  }
  if (c->mode == SIF_MODE_FIXED &&
      check_cuda(cudaMemcpyAsync(wb + w.fixedq, c->fixed_q, (size_t)(c->m_plus + c->m_minus), cudaMemcpyHostToDevice, s)))
    return SIF_ERR_CUDA;
  // digit histograms start zeroed; enc_select re-zeroes each one after reading it
  if (p->cap_smem > 0 &&
      check_cuda(cudaMemsetAsync(wb + w.hist, 0, 4ull * 2 * sif::ND * (uint64_t)p->cap_smem, s)))
    return SIF_ERR_CUDA;
  // the uploads read host vectors: finish them before the vectors go out of scope
  return check_cuda(cudaStreamSynchronize(s));
}

static int enc_launch(const sif_plan* p, const sif_codec_cfg* c, void* ws, uint64_t* out_len, int32_t* status,
                      int atkf, int64_t* kept, double* tau3, cudaStream_t s) {
  if (p->n == 0) return SIF_OK;
  uint8_t* wb = (uint8_t*)ws;
  const EncWs w = enc_ws(p->n, (uint64_t)p->tiles, p->max_blocks, (uint64_t)p->cap_smem, (uint64_t)c->m_plus + c->m_minus);
  sif::EArgs a;
  memset(&a, 0, sizeof(a));
  a.info = reinterpret_cast<const sif::IfInfo*>(wb + w.info);
  a.st = reinterpret_cast<sif::IfSt*>(wb + w.st);
  a.n = p->n;
  a.nch = p->tiles;
  a.maxb = p->max_blocks;
  a.atkf_only = atkf;
  a.ch_if = reinterpret_cast<const uint32_t*>(wb + w.ch_if);
  a.ch_e0 = reinterpret_cast<const uint32_t*>(wb + w.ch_e0);
  a.u_off = reinterpret_cast<uint32_t*>(wb + w.u_off);
  a.u_cnt = reinterpret_cast<uint32_t*>(wb + w.u_cnt);
  a.seg_base = reinterpret_cast<const uint32_t*>(wb + w.segbase);
  a.ch_bcnt = reinterpret_cast<uint32_t*>(wb + w.bcnt);
  a.ch_bpre = reinterpret_cast<uint32_t*>(wb + w.bpre);
  a.ch_brs = reinterpret_cast<uint32_t*>(wb + w.brs);
  a.ch_blast = reinterpret_cast<int32_t*>(wb + w.blast);
  a.ch_bprev = reinterpret_cast<int32_t*>(wb + w.bprev);
  a.hist = reinterpret_cast<uint32_t*>(wb + w.hist);
  a.big_list = reinterpret_cast<uint32_t*>(wb + w.biglist);
  a.inject = getenv("SIF_TEST_INJECT") ? (uint32_t)atoi(getenv("SIF_TEST_INJECT")) : 0u;  // tests only
  a.ws = wb;
  a.s = c->s; a.lam = c->lam; a.delta = c->delta;
  a.m_plus = c->m_plus; a.m_minus = c->m_minus; a.q_bit = c->q_bit; a.mode = c->mode;
  a.fixed_q = wb + w.fixedq;
  a.out_len = out_len;
  a.status = status;
  a.kept_out = kept;
  a.kept_off = reinterpret_cast<const uint64_t*>(wb + w.keptoff);
  a.tau3 = tau3;
  // multi-kernel select for IFs with many candidates (one CTA per IF would scan them
  // alone); enabled when the batch holds an IF whose keep count exceeds half the cut-off
  a.big_ncand = (p->flags & 2) ? big_ncand() : 0u;
  a.prof = reinterpret_cast<uint64_t*>(getenv("SIF_PROF_PTR") ? strtoull(getenv("SIF_PROF_PTR"), nullptr, 0) : 0ull);
  DevState* ds = dev_state();
  if (!ds) return SIF_ERR_CUDA;
  const int maxb = p->max_blocks;
  int g_abq, g_pack;
  {
    std::lock_guard<std::mutex> lk(ds->mu);
    if (!ds->g_abq[maxb]) {
      ds->g_abq[maxb] = maxb > 32 ? resident_grid(sif::enc_abq<1, true>, sif::CNT, smem_abq(maxb), 1ull << 30, ds->sms)
                                  : resident_grid(sif::enc_abq<1, false>, sif::CNT, smem_abq(maxb), 1ull << 30, ds->sms);
      ds->g_pack[maxb] = maxb > 32 ? resident_grid(sif::enc_pack<true>, sif::CNT, smem_pack(maxb), 1ull << 30, ds->sms)
                                   : resident_grid(sif::enc_pack<false>, sif::CNT, smem_pack(maxb), 1ull << 30, ds->sms);
    }
    g_abq = ds->g_abq[maxb];
    g_pack = ds->g_pack[maxb];
  }
  const int g_stream = ds->g_stream, g_members = ds->g_members, g_gather = ds->g_gather, g_crc = ds->g_crc;
  const unsigned nch = (unsigned)p->tiles;
  const unsigned n = (unsigned)p->n;
  const unsigned wgrid = std::max(1u, (nch + sif::CNT / 32 - 1) / (sif::CNT / 32));  // >= 1 chunk per warp
  if (p->reserved > 0) {
    ProfScope ps(KP_TOKEN, s);
    sif::enc_token<<<(unsigned)p->reserved, sif::KNT, 0, s>>>(a, reinterpret_cast<const uint32_t*>(wb + w.tokens));
  }
  if (p->reserved == p->n) return check_cuda(cudaGetLastError());
  {
    ProfScope ps(KP_PREP, s);
    if (p->flags & 8) sif::enc_prep<128, true><<<n, 128, 0, s>>>(a);  // every IF fits one chunk
    else sif::enc_prep<512, false><<<n, 512, 0, s>>>(a);
  }
  { ProfScope ps(KP_STREAM, s); sif::enc_stream<<<std::min<unsigned>(nch, g_stream), sif::CNT, kSmemStream, s>>>(a); }
  if (p->n_fused > 0) {
    ProfScope ps(KP_FUSED, s);
    sif::enc_post<<<(unsigned)p->n_fused, sif::PNT, ds->post_smem, s>>>(a, reinterpret_cast<const uint32_t*>(wb + w.fused),
                                                                        ds->post_lcap);
  }
  if (p->n_fused == p->n) return check_cuda(cudaGetLastError());
  if (p->flags & 4) {
    ProfScope ps(KP_SELECT_TINY, s);
    sif::enc_select_tiny<<<(n + sif::TNT / 32 - 1) / (sif::TNT / 32), sif::TNT, 0, s>>>(a);
  }
  {
    // lambda > 0 with IFs on the multi-kernel path: their tau / class / kept-count passes run
    // in enc_select<0>, deeper load pipelining measured faster there (C4 lambda = 0.1:
    // 1967 -> 1710 us) and slower for small IFs (C2: 64 -> 110 us)
    ProfScope ps(KP_SELECT, s);
    if (a.big_ncand && c->lam > 0.0) sif::enc_select<0, true><<<n, sif::SNT, kSmemSelect, s>>>(a);
    else if (c->lam > 0.0 || atkf) sif::enc_select<0><<<n, sif::SNT, kSmemSelect, s>>>(a);
    else sif::enc_select<0, false, true><<<n, sif::SNT, kSmemSelect, s>>>(a);  // lambda = 0 encode
  }
  if (a.big_ncand) {  // some IF is large enough for the multi-kernel select
    { ProfScope ps(KP_GATHER1, s); sif::enc_gather<1><<<std::min<unsigned>(wgrid, g_gather), sif::CNT, 0, s>>>(a); }
    {
      ProfScope ps(KP_SELECT1, s);
      if (c->lam > 0.0 || atkf) sif::enc_select<1><<<n, sif::SNT, kSmemSelect, s>>>(a);
      else sif::enc_select<1, false, true><<<n, sif::SNT, kSmemSelect, s>>>(a);  // lambda = 0 encode
    }
    if (!atkf) {
      { ProfScope ps(KP_GATHER2, s); sif::enc_gather<2><<<std::min<unsigned>(wgrid, g_gather), sif::CNT, 0, s>>>(a); }
      {
        ProfScope ps(KP_SELECT2, s);
        const dim3 g2(n, (unsigned)std::max(1, std::min(maxb - 2, 8)));  // one CTA per pending cut
        sif::enc_select<2><<<g2, sif::SNT, kSmemSelect, s>>>(a);
      }
    }
  }
  if (!atkf) {
    { ProfScope ps(KP_MEMBERS, s); sif::enc_members<<<std::min<unsigned>(wgrid, g_members), sif::CNT, 0, s>>>(a); }
    if (c->mode != SIF_MODE_FIXED) {
      const unsigned ga = std::min<unsigned>(wgrid, g_abq);
      if (maxb > 32) {
        { ProfScope ps(KP_ABQ1, s); sif::enc_abq<1, true><<<ga, sif::CNT, smem_abq(maxb), s>>>(a); }
        { ProfScope ps(KP_ABQ2, s); sif::enc_abq<0, true><<<ga, sif::CNT, smem_abq(maxb), s>>>(a); }
      } else {
        { ProfScope ps(KP_ABQ1, s); sif::enc_abq<1, false><<<ga, sif::CNT, smem_abq(maxb), s>>>(a); }
        { ProfScope ps(KP_ABQ2, s); sif::enc_abq<0, false><<<ga, sif::CNT, smem_abq(maxb), s>>>(a); }
      }
    }
    { ProfScope ps(KP_LAYOUT, s); sif::enc_layout<<<n, 256, 0, s>>>(a); }
    {
      ProfScope ps(KP_PACK, s);
      if (maxb > 32) sif::enc_pack<true><<<std::min<unsigned>(wgrid, g_pack), sif::CNT, smem_pack(maxb), s>>>(a);
      else sif::enc_pack<false><<<std::min<unsigned>(wgrid, g_pack), sif::CNT, smem_pack(maxb), s>>>(a);
    }
    { ProfScope ps(KP_CRC, s); sif::enc_crc<<<std::min<unsigned>((unsigned)p->cluster, g_crc), sif::CNT, 0, s>>>(a); }
  }
  return check_cuda(cudaGetLastError());
}

int sif_enc_run(const sif_plan* p, const sif_codec_cfg* c, void* ws, uint64_t* out_len, int32_t* status, void* stream) {
  if (!p || !c || !ws || !out_len || !status) return SIF_ERR_INVALID_ARG;
  if (p->flags & 1) return SIF_ERR_INVALID_ARG;  // an ATKF-only plan
  return enc_launch(p, c, ws, out_len, status, 0, nullptr, nullptr, (cudaStream_t)stream);
}

int sif_encode_batched(const sif_enc_desc* d, int n, const sif_codec_cfg* c, void* ws, size_t ws_bytes,
                       uint64_t* out_len, int32_t* status, void* stream) {
  sif_plan p;
  int st = sif_enc_plan(d, n, c, &p);
  if (st) return st;
  if (ws_bytes < p.ws_bytes) return SIF_ERR_CAPACITY;
  st = sif_enc_upload(&p, d, c, ws, stream);
  if (st) return st;
  return sif_enc_run(&p, c, ws, out_len, status, stream);
}

int sif_atkf_batched(const sif_enc_desc* d, int n, const sif_codec_cfg* c, void* ws, size_t ws_bytes, int64_t* kept,
                     double* tau3, int32_t* status, void* stream) {
  sif_plan p;
  int st = enc_plan_impl(d, n, c, 1, &p);
  if (st) return st;
  if (ws_bytes < p.ws_bytes) return SIF_ERR_CAPACITY;
  cudaStream_t s = (cudaStream_t)stream;
  st = sif_enc_upload(&p, d, c, ws, stream);
  if (st) return st;
  std::vector<uint64_t> off((size_t)std::max(n, 1), 0);
  uint64_t acc = 0;
  for (int i = 0; i < n; ++i) {
    off[i] = acc;
    acc += sif::keep_count(c->s, (uint64_t)d[i].rows * d[i].cols);
  }
  const EncWs w = enc_ws(p.n, (uint64_t)p.tiles, p.max_blocks, (uint64_t)p.cap_smem, (uint64_t)c->m_plus + c->m_minus);
  if (n > 0 && check_cuda(cudaMemcpyAsync((uint8_t*)ws + w.keptoff, off.data(), 8ull * n, cudaMemcpyHostToDevice, s)))
    return SIF_ERR_CUDA;
  st = enc_launch(&p, c, ws, nullptr, status, 1, kept, tau3, s);
  if (st) return st;
  return check_cuda(cudaStreamSynchronize(s));
}

// ------------------------------------------------------------------ decode
static uint32_t dec_segments(uint64_t len) {
  const uint64_t body = len > 8 ? len - 8 : 0;  // CRC range [4, len - 4)
  return (uint32_t)std::max<uint64_t>(1, (body + sif::SEGD - 1) / sif::SEGD);
}

// Table rows of one stream: 2 header rows + one per block.  A block takes at least
// 13 + 4 (rows + 1) bytes (codec.py:303-315), so a stream of in_len bytes (or capacity)
// holds at most (in_len - 36) / that many blocks; at most 2 * 65535 (u16 M+ / M-).
static uint64_t dec_table_rows(const sif_dec_desc& d) {
  const uint64_t per = 13ull + 4ull * ((uint64_t)d.rows + 1);
  const uint64_t body = d.in_len > 36 ? d.in_len - 36 : 0;
  return 2 + std::min<uint64_t>(body / per + 1, 2ull * 65535);
}

struct DecWs {
  uint64_t desc, table, taboff, acc, segbase, itembase, small, slist, total;
};

// Streams decoded by sif_dec_small (one CTA each): the dense output fits in shared memory.
static std::atomic<uint64_t> g_small_max{sif::SMALL_T};
static bool dec_is_small(const sif_dec_desc& d) {
  return d.rows >= 1 && d.cols >= 1 && (uint64_t)d.rows * d.cols <= g_small_max.load(std::memory_order_relaxed);
}

int sif_set_small_decode(uint64_t max_elems) {
  if (max_elems > sif::SMALL_T) return SIF_ERR_INVALID_ARG;
  g_small_max.store(max_elems);
  g_routing_epoch.fetch_add(1);
  return SIF_OK;
}

static DecWs dec_ws(uint64_t n, uint64_t table_rows) {
  DecWs w;
  uint64_t off = 0;
  auto take = [&](uint64_t bytes) { const uint64_t o = off; off += up(std::max<uint64_t>(bytes, 1), 256); return o; };
  w.desc = take(sizeof(sif_dec_desc) * n);
  w.table = take(table_rows * 64ull);
  w.taboff = take(8ull * (n + 1));
  w.acc = take(16ull * n);
  w.segbase = take(4ull * (n + 1));
  w.itembase = take(8ull * (n + 1));
  w.small = take(4ull * n);
  w.slist = take(4ull * n);
  w.total = off;
  return w;
}

// Elements per decode work item: a group of whole rows, or a segment of one long row.
// Batches of narrow IFs (every K <= 1280) take 1280-element row groups (small items keep
// the warps balanced); wider rows take 4096-element items (a 4096-column row is one item,
// no column-segment searches).  The scatter keeps only two bitmaps per item in shared
// memory (the output is written in place), so the item size is free.
static uint32_t dec_segw(const sif_dec_desc* d, int n) {
  for (int i = 0; i < n; ++i)
    if (d[i].cols > 1280 && !dec_is_small(d[i])) return 4096;
  return 1280;
}

int sif_dec_plan(const sif_dec_desc* d, int n, sif_plan* p) {
  if (!p || (n > 0 && !d) || n < 0) return SIF_ERR_INVALID_ARG;
  memset(p, 0, sizeof(*p));
  uint64_t rows = 0, nseg = 0;
  int nsmall = 0;
  for (int i = 0; i < n; ++i) {
    if (!d[i].in || (reinterpret_cast<uintptr_t>(d[i].in) & 3)) return SIF_ERR_INVALID_ARG;
    if (d[i].in_len_dev && (reinterpret_cast<uintptr_t>(d[i].in_len_dev) & 7)) return SIF_ERR_INVALID_ARG;
    rows += dec_table_rows(d[i]);
    if (dec_is_small(d[i])) { ++nsmall; continue; }
    nseg += dec_segments(d[i].in_len);
    if (dec_segments(d[i].in_len) > (uint32_t)sif::CRC_PIECES_MAX) return SIF_ERR_INVALID_ARG;
  }
  if (nseg >= (1ull << 31)) return SIF_ERR_INVALID_ARG;
  const uint32_t segw = dec_segw(d, n);
  p->n = n;
  p->threads = sif::DNT;
  p->tiles = (int32_t)segw;    // decode plans: columns per work item
  p->cluster = (int32_t)nseg;  // decode plans: CRC segment CTAs
  p->max_blocks = 0;
  p->smem_bytes = (sif::DNT / 32) * (int)(2 * ((segw + 31) / 32) * 4);
  const DecWs w = dec_ws(std::max(n, 1), rows);
  p->ws_desc_off = w.desc;
  p->ws_aux_off = w.table;
  p->ws_spill_off = rows;  // decode plans: total table rows
  p->ws_bytes = w.total;
  p->n_fused = nsmall;     // decode plans: streams on the small-stream kernel
  return SIF_OK;
}

uint64_t sif_dec_table_offset(const sif_plan* p, const sif_dec_desc* d, int i) {
  if (!p || !d || i < 0 || i >= p->n) return 0;
  uint64_t rows = 0;
  for (int k = 0; k < i; ++k) rows += dec_table_rows(d[k]);
  return p->ws_aux_off + 64ull * rows;
}

int sif_dec_upload(const sif_plan* p, const sif_dec_desc* d, void* ws, void* stream) {
  if (!p || !ws) return SIF_ERR_INVALID_ARG;
  if (!dev_state()) return SIF_ERR_CUDA;
  cudaStream_t s = (cudaStream_t)stream;
  uint8_t* wb = (uint8_t*)ws;
  if (p->n == 0) return SIF_OK;
  const DecWs w = dec_ws(p->n, p->ws_spill_off);
  if (check_cuda(cudaMemcpyAsync(wb + w.desc, d, sizeof(sif_dec_desc) * p->n, cudaMemcpyHostToDevice, s)))
    return SIF_ERR_CUDA;
  const uint32_t segw = (uint32_t)p->tiles;
  std::vector<uint32_t> seg((size_t)p->n + 1, 0);
  std::vector<uint64_t> items((size_t)p->n + 1, 0), toff((size_t)p->n + 1, 0);
  std::vector<uint32_t> small((size_t)p->n, 0), slist;
  for (int i = 0; i < p->n; ++i) {
    toff[i + 1] = toff[i] + dec_table_rows(d[i]) * sif::TROW_U32;
    if (dec_is_small(d[i])) {  // no CRC pieces / work items on the four-kernel path
      small[i] = 1;
      slist.push_back((uint32_t)i);
      seg[i + 1] = seg[i];
      items[i + 1] = items[i];
      continue;
    }
    seg[i + 1] = seg[i] + dec_segments(d[i].in_len);
    const uint32_t R = d[i].cols <= segw && d[i].cols ? segw / d[i].cols : 1u;  // rows per item
    items[i + 1] = items[i] + (uint64_t)((d[i].rows + R - 1) / R) * ((d[i].cols + segw - 1) / segw);
  }
  if (check_cuda(cudaMemcpyAsync(wb + w.small, small.data(), 4ull * p->n, cudaMemcpyHostToDevice, s)))
    return SIF_ERR_CUDA;
  if (!slist.empty() &&
      check_cuda(cudaMemcpyAsync(wb + w.slist, slist.data(), 4ull * slist.size(), cudaMemcpyHostToDevice, s)))
    return SIF_ERR_CUDA;
  if (check_cuda(cudaMemsetAsync(wb + w.acc, 0, 16ull * p->n, s))) return SIF_ERR_CUDA;
  // the table's unused words are read back by the host with each row: start them at zero
  if (check_cuda(cudaMemsetAsync(wb + w.table, 0, 64ull * p->ws_spill_off, s))) return SIF_ERR_CUDA;
  if (check_cuda(cudaMemcpyAsync(wb + w.segbase, seg.data(), 4ull * (p->n + 1), cudaMemcpyHostToDevice, s)))
    return SIF_ERR_CUDA;
  if (check_cuda(cudaMemcpyAsync(wb + w.itembase, items.data(), 8ull * (p->n + 1), cudaMemcpyHostToDevice, s)))
    return SIF_ERR_CUDA;
  if (check_cuda(cudaMemcpyAsync(wb + w.taboff, toff.data(), 8ull * (p->n + 1), cudaMemcpyHostToDevice, s)))
    return SIF_ERR_CUDA;
  return check_cuda(cudaStreamSynchronize(s));
}

int sif_dec_run(const sif_plan* p, int parse_only, void* ws, int32_t* status, void* stream) {
  if (!p || !ws || !status) return SIF_ERR_INVALID_ARG;
  if (p->n == 0) return SIF_OK;
  DevState* ds = dev_state();
  if (!ds) return SIF_ERR_CUDA;
  cudaStream_t s = (cudaStream_t)stream;
  uint8_t* wb = (uint8_t*)ws;
  const DecWs w = dec_ws(p->n, p->ws_spill_off);
  sif::DecArgs a;
  memset(&a, 0, sizeof(a));
  a.descs = reinterpret_cast<const sif_dec_desc*>(wb + w.desc);
  a.n = p->n;
  a.table = reinterpret_cast<uint32_t*>(wb + w.table);
  a.tab_off = reinterpret_cast<const uint64_t*>(wb + w.taboff);
  a.acc = reinterpret_cast<uint32_t*>(wb + w.acc);
  a.parse_only = parse_only;
  a.status = status;
  a.seg_base = reinterpret_cast<const uint32_t*>(wb + w.segbase);
  a.item_base = reinterpret_cast<const uint64_t*>(wb + w.itembase);
  a.segw = p->tiles;
  a.small = reinterpret_cast<const uint32_t*>(wb + w.small);
  a.small_list = reinterpret_cast<const uint32_t*>(wb + w.slist);
  if (p->n_fused > 0) {
    ProfScope ps(KP_DSMALL, s);
    sif::sif_dec_small<<<(unsigned)p->n_fused, sif::DSN, 0, s>>>(a);
  }
  if (p->n_fused == p->n) return check_cuda(cudaGetLastError());
  { ProfScope ps(KP_PARSE, s); sif::sif_parse_kernel<<<(p->n + 127) / 128, 128, 0, s>>>(a); }
  {
    const unsigned warps = (unsigned)p->cluster;
    const unsigned grid = std::min<unsigned>((warps + sif::DNT / 32 - 1) / (sif::DNT / 32), ds->g_dcrc);
    ProfScope ps(KP_DCRC, s);
    sif::sif_dcrc_kernel<<<std::max(1u, grid), sif::DNT, 0, s>>>(a);
  }
  if (!parse_only) {
    int per = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, sif::sif_scatter_kernel, sif::DNT, p->smem_bytes) != cudaSuccess ||
        per < 1)
      per = 1;
    ProfScope ps(KP_SCATTER, s);
    sif::sif_scatter_kernel<<<(unsigned)(per * ds->sms), sif::DNT, p->smem_bytes, s>>>(a);
  }
  { ProfScope ps(KP_DFINAL, s); sif::sif_dfinal_kernel<<<(p->n + 127) / 128, 128, 0, s>>>(a); }
  return check_cuda(cudaGetLastError());
}

int sif_decode_batched(const sif_dec_desc* d, int n, int parse_only, void* ws, size_t ws_bytes, int32_t* status,
                       void* stream) {
  sif_plan p;
  int st = sif_dec_plan(d, n, &p);
  if (st) return st;
  if (ws_bytes < p.ws_bytes) return SIF_ERR_CAPACITY;
  st = sif_dec_upload(&p, d, ws, stream);
  if (st) return st;
  return sif_dec_run(&p, parse_only, ws, status, stream);
}

// ------------------------------------------------------------------ input rebinding
// A plan's descriptors live in its workspace; these rebind one IF's / stream's buffers on
// the device (a one-thread kernel: stream-ordered, no host synchronisation), so a cached
// plan serves a new call with the same shapes (the single-IF encode() / decode() API).
int sif_enc_set_input(const sif_plan* p, void* ws, int i, const void* x, uint8_t* out, uint64_t seed, void* stream) {
  if (!p || !ws || i < 0 || i >= p->n || !x || (reinterpret_cast<uintptr_t>(x) & 15) || !out ||
      (reinterpret_cast<uintptr_t>(out) & 15))
    return SIF_ERR_INVALID_ARG;
  sif::IfInfo* info = reinterpret_cast<sif::IfInfo*>((uint8_t*)ws + p->ws_desc_off) + i;
  sif::set_enc_input_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(info, x, out, seed);
  return check_cuda(cudaGetLastError());
}

int sif_dec_set_input(const sif_plan* p, void* ws, int i, const uint8_t* in, uint64_t len, uint64_t* d_len_slot,
                      float* out, void* stream) {
  if (!p || !ws || i < 0 || i >= p->n || !in || (reinterpret_cast<uintptr_t>(in) & 3) || !d_len_slot ||
      (reinterpret_cast<uintptr_t>(d_len_slot) & 7) || !out)
    return SIF_ERR_INVALID_ARG;
  sif_dec_desc* d = reinterpret_cast<sif_dec_desc*>((uint8_t*)ws + p->ws_desc_off) + i;
  sif::set_dec_input_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(d, in, d_len_slot, len, out);
  return check_cuda(cudaGetLastError());
}

// ------------------------------------------------------------------ synthetic inputs
int sif_gen_synthetic(void* x, uint32_t rows, uint32_t cols, uint32_t dtype, uint32_t kind, uint64_t sid, void* stream) {
  if (!x || rows == 0 || cols == 0) return SIF_ERR_INVALID_ARG;
  const uint64_t T = (uint64_t)rows * cols;
  const unsigned grid = (unsigned)std::min<uint64_t>((T + 255) / 256, 148ull * 16);
  sif::sif_synth_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(x, rows, cols, dtype, kind, sid);
  return check_cuda(cudaGetLastError());
}

int sif_fixture_tensor(float* x, uint64_t n, uint64_t seed, int dist, void* stream) {
  if ((!x && n) || (dist != 0 && dist != 1)) return SIF_ERR_INVALID_ARG;
  if (n == 0) return SIF_OK;
  const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 16);
  sif::sif_fixture_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(x, n, seed, (uint32_t)dist);
  return check_cuda(cudaGetLastError());
}

int sif_count_nonfinite(const float* x, uint64_t n, unsigned long long* d_count, void* stream) {
  if ((!x && n) || !d_count || (reinterpret_cast<uintptr_t>(x) & 15)) return SIF_ERR_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (check_cuda(cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), s))) return SIF_ERR_CUDA;
  if (n == 0) return SIF_OK;
  const unsigned grid = (unsigned)std::min<uint64_t>((n / 4 + 255) / 256 + 1, 148ull * 8);
  sif::sif_nonfinite_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const uint32_t*>(x), n, d_count);
  return check_cuda(cudaGetLastError());
}

}  // extern "C"
