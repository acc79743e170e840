/*
 * sif.h -- C ABI of the B200-native SLICER intermediate-feature (IF) codec.
 *
 * This is the drop-in boundary for the reference codec path
 * (/root/reference/pkg/src/slicer/codec.py).  The reference has no FFI: its boundary is
 * the Python API re-exported at __init__.py:15-25.  Each entry point below replaces one
 * (or a fused pair) of those calls; the Python mirror in paper_2511_11608_b200/codec.py
 * keeps the reference names and raises the reference exception classes from the status
 * codes.  Plain pointers and sizes only; all buffers are caller-owned device memory;
 * nothing is allocated per call; every call is stream-ordered and asynchronous.
 *
 *   reference call                                   replaced by
 *   ------------------------------------------------ -----------------------------------
 *   serialize(encode(x, cfg, seed))  codec.py:186,:283  sif_encode_batched / sif_enc_*
 *   decode(deserialize(data))        codec.py:320,:254  sif_decode_batched / sif_dec_*
 *   deserialize(data) (checks only)  codec.py:320-385   sif_decode_batched(..., parse_only=1)
 *   atkf_filter(x, s, lam, seed)     atkf.py:44-96      sif_atkf_batched
 *   payload_upper_bound (capacity)   planner.py:33-64   sif_max_payload_bytes (sound for fixed q)
 *   keep_count / col_bits            atkf.py:31, codec.py:57   sif_keep_count / sif_col_bits
 */
#ifndef SIF_H_
#define SIF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: 1:1 with the reference exception classes (errors.py:4-37). */
enum sif_status {
  SIF_OK = 0,
  SIF_ERR_CONFIG = 1,         /* ConfigError        codec.py:72-92, atkf.py:45-48          */
  SIF_ERR_NONFINITE = 2,      /* NonFiniteError     atkf.py:50-51, tensor.py:35-36         */
  SIF_ERR_SHAPE = 3,          /* ShapeError         tensor.py:27-33                        */
  SIF_ERR_STREAM_FORMAT = 4,  /* StreamFormatError  codec.py:321-385                       */
  SIF_ERR_CORRUPT_STREAM = 5, /* CorruptStreamError codec.py:235-252, :351-352             */
  SIF_ERR_CAPACITY = 6,       /* caller buffer too small / shape mismatch (no ref analogue) */
  SIF_ERR_CUDA = 7,           /* CUDA launch/runtime failure                               */
  SIF_ERR_INVALID_ARG = 8     /* bad pointer/size at the ABI (no ref analogue)             */
};

enum { SIF_DTYPE_F32 = 0, SIF_DTYPE_BF16 = 1 };
enum { SIF_MODE_ABQ = 0, SIF_MODE_FIXED = 1 };

/* Effective blocks (min(M+, k) + min(M-, k), msplit.py:34-38) per IF the encoder supports;
 * sif_enc_plan returns SIF_ERR_CONFIG above it (the reference has no limit). */
#define SIF_MAX_BLOCKS 64

/* CodecConfig (codec.py:61-92).  fixed_q is a HOST pointer with m_plus+m_minus entries
 * (plus-plane entries first), read only during sif_enc_upload / sif_encode_batched. */
typedef struct sif_codec_cfg {
  double s;
  double lam;
  double delta;
  int32_t m_plus;
  int32_t m_minus;
  int32_t q_bit;
  int32_t mode;
  const uint8_t* fixed_q;
} sif_codec_cfg;

/* One IF to encode: x is rows x cols row-major on the device (fp32 or bf16); out is a
 * device buffer of out_cap bytes, 16-byte aligned (>= sif_max_payload_bytes). */
typedef struct sif_enc_desc {
  const void* x;
  uint8_t* out;
  uint64_t out_cap;
  uint64_t seed;
  uint32_t rows;
  uint32_t cols;
  uint32_t dtype;
  uint32_t reserved;
} sif_enc_desc;

/* One .sif stream to decode into a dense fp32 rows x cols tensor.  `in` is 4-byte
 * aligned device memory; rows/cols must match the stream header.
 * in_len_dev == NULL: the stream is in_len bytes long.
 * in_len_dev != NULL: in_len is the capacity of `in` and the stream length is read ON THE
 * DEVICE from *in_len_dev when the decode runs -- point it at the encoder's d_out_len[i]
 * so a plan (or a captured CUDA graph) of encode -> decode stays valid when the inputs,
 * and therefore the payload lengths, change from one run to the next. */
typedef struct sif_dec_desc {
  const uint8_t* in;
  uint64_t in_len;
  float* out;
  uint32_t rows;
  uint32_t cols;
  const uint64_t* in_len_dev;
} sif_dec_desc;

/* Launch plan for a batch (host-only computation, POD). */
typedef struct sif_plan {
  int32_t n;            /* IFs in the batch                                 */
  int32_t cluster;      /* CTAs cooperating on one IF (thread-block cluster) */
  int32_t threads;      /* threads per CTA                                  */
  int32_t smem_bytes;   /* dynamic shared memory per CTA                    */
  int32_t cap_smem;     /* list entries held in shared memory per CTA       */
  int32_t max_blocks;   /* M+ + M- upper bound                              */
  int32_t tiles;        /* decode: row-slab tiles in the grid               */
  int32_t flags;
  uint64_t ws_bytes;    /* device workspace required                        */
  uint64_t ws_desc_off; /* offsets of the sections inside the workspace     */
  uint64_t ws_aux_off;
  uint64_t ws_spill_off;
  int32_t n_fused;      /* encode: IFs finished by the per-IF back end          */
  int32_t reserved;     /* encode: IFs on the token path (one CTA each)         */
} sif_plan;

/* ---- scalars (host) ---- */
uint64_t sif_keep_count(double s, uint64_t t);                     /* atkf.py:31-34   */
uint32_t sif_col_bits(uint32_t k);                                 /* codec.py:57-58  */
int sif_validate_cfg(const sif_codec_cfg* cfg);                    /* codec.py:72-92  */
uint64_t sif_max_payload_bytes(uint32_t rows, uint32_t cols, const sif_codec_cfg* cfg);
const char* sif_status_string(int status);
int sif_version(void);

/* ---- encode: encode + serialize (codec.py:186-232, :283-317) ----
 * sif_enc_plan: host-only.  sif_enc_upload: stream-ordered copy of the descriptors and
 * config into the workspace (do once per batch layout).  sif_enc_run: launches only
 * (graph-capturable).  Per IF, out_len[i] = exact .sif length and status[i] a sif_status. */
int sif_enc_plan(const sif_enc_desc* descs, int n, const sif_codec_cfg* cfg, sif_plan* plan);
int sif_enc_upload(const sif_plan* plan, const sif_enc_desc* descs, const sif_codec_cfg* cfg,
                   void* d_ws, void* stream);
int sif_enc_run(const sif_plan* plan, const sif_codec_cfg* cfg, void* d_ws, uint64_t* d_out_len,
                int32_t* d_status, void* stream);
/* Size classes: multi-chunk IFs of tmin..tmax elements (default: none) finish their encode
 * in the per-IF back end (one CTA per IF after the stream pass), all others in the chunk
 * pipeline; both produce the same bytes.  Process-wide, read by sif_enc_plan (a plan keeps
 * the routing it was made with). */
int sif_set_fused_range(uint64_t tmin, uint64_t tmax);
int sif_get_fused_range(uint64_t* tmin, uint64_t* tmax);
/* plan + upload + run in one call. */
int sif_encode_batched(const sif_enc_desc* descs, int n, const sif_codec_cfg* cfg, void* d_ws,
                       size_t ws_bytes, uint64_t* d_out_len, int32_t* d_status, void* stream);

/* ---- ATKF only (atkf.py:44-96): kept flat indices (ascending) and tau ----
 * d_kept holds the concatenation over IFs (in batch order) of keep_count(s, rows*cols)
 * int64 entries each; d_tau3[3*i .. 3*i+2] = {tau, tau_plus, tau_minus}. */
int sif_atkf_batched(const sif_enc_desc* descs, int n, const sif_codec_cfg* cfg, void* d_ws,
                     size_t ws_bytes, int64_t* d_kept, double* d_tau3, int32_t* d_status,
                     void* stream);

/* ---- decode: deserialize + decode (codec.py:320-399, :235-266) ----
 * parse_only=1 stops after the deserialize checks (magic, CRC, version, mode, framing, q
 * range) and fills the block table; otherwise the dense fp32 outputs are written too. */
int sif_dec_plan(const sif_dec_desc* descs, int n, sif_plan* plan);
int sif_dec_upload(const sif_plan* plan, const sif_dec_desc* descs, void* d_ws, void* stream);
int sif_dec_run(const sif_plan* plan, int parse_only, void* d_ws, int32_t* d_status, void* stream);
int sif_decode_batched(const sif_dec_desc* descs, int n, int parse_only, void* d_ws,
                       size_t ws_bytes, int32_t* d_status, void* stream);
/* Rebind one IF / stream of an uploaded plan to new device buffers (stream-ordered, no host
 * synchronisation): a cached plan then serves a new call with the same shapes and config.
 * Encode: x and out as in sif_enc_desc (16-byte aligned; out of the plan's capacity), seed.
 * Decode (the plan must have been made with the stream's CAPACITY as in_len): in (4-byte
 * aligned), its length len (<= that capacity; written to the device slot d_len_slot, which
 * becomes the descriptor's in_len_dev), out (rows x cols fp32). */
int sif_enc_set_input(const sif_plan* plan, void* d_ws, int i, const void* d_x, uint8_t* d_out,
                      uint64_t seed, void* stream);
int sif_dec_set_input(const sif_plan* plan, void* d_ws, int i, const uint8_t* d_in, uint64_t len,
                      uint64_t* d_len_slot, float* d_out, void* stream);

/* Size class: streams of at most max_elems dense elements (default and maximum 4096; 0 =
 * none) are decoded by one CTA each in a single launch (the stream staged in shared
 * memory), the others by the four-kernel path; both give the same output, status and
 * block table.  Process-wide, read by sif_dec_plan (a plan keeps its routing). */
int sif_set_small_decode(uint64_t max_elems);
/* Incremented by sif_set_fused_range / sif_set_small_decode: callers that cache plans key
 * them on it so a routing change takes effect on the next call. */
uint64_t sif_routing_epoch(void);

/* Block table written by decode/parse: 64-byte rows of uint32.  Row 0 holds {status,
 * rows, cols, m_plus, m_minus, mode, q_bit, nblocks}; row 1 {framing status, crc, len lo,
 * len hi, reasons...}; then one row per block (plus blocks first) {q, nnz, o_bits,
 * vmin_bits, rowptr_off (u64), cols_off (u64), codes_off (u64)}.  Stream i's table starts
 * sif_dec_table_offset(plan, descs, i) bytes into d_ws (descs as passed to sif_dec_plan). */
uint64_t sif_dec_table_offset(const sif_plan* plan, const sif_dec_desc* descs, int i);

/* ---- per-kernel timing (diagnostics) ----
 * While enabled, every kernel launched by sif_enc_run / sif_dec_run is bracketed by CUDA
 * events on its stream.  sif_profile_read synchronizes those events, fills ms[k] (total
 * milliseconds) and count[k] (launches) for kernel kinds k < maxk, clears the record and
 * returns the number of kernel kinds (or -status on failure); sif_profile_kernel_name(k)
 * names kind k. */
int sif_profile_enable(int on);
int sif_profile_enabled(void); /* 1 while enabled (graph-replayed calls bypass the brackets) */
int sif_profile_read(double* ms, int32_t* count, int maxk);
const char* sif_profile_kernel_name(int k);

/* ---- device synthetic IF generator (bench/tests) ---- */
int sif_gen_synthetic(void* d_x, uint32_t rows, uint32_t cols, uint32_t dtype, uint32_t kind,
                      uint64_t sid, void* stream);

/* ---- fixture tensors and .tns validation ----
 * sif_fixture_tensor: random_tensor(rows, cols, seed, dist) values (tensor.py:90-111,
 * rng.py:30-52) for n = rows*cols fp32 elements; dist 0 = "uniform" (bit-identical),
 * 1 = "gaussian" (CUDA log/sin/cos; see sif_synth.cu).
 * sif_count_nonfinite: number of NaN/Inf elements of x into *d_count (device u64), the
 * finiteness check of load_tensor / DenseTensor (tensor.py:35-36, :84-85). */
int sif_fixture_tensor(float* d_x, uint64_t n, uint64_t seed, int dist, void* stream);
int sif_count_nonfinite(const float* d_x, uint64_t n, unsigned long long* d_count, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SIF_H_ */
