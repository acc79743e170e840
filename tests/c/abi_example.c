/* abi_example.c -- a plain C caller of the codec's C ABI (include/sif.h), the binding a
 * maintainer would write.  One-call entry points only:
 *   sif_encode_batched  == serialize(encode(x, cfg, seed))   codec.py:186, :283
 *   sif_decode_batched  == decode(deserialize(data))         codec.py:320, :254
 * Encodes (1) the 1x6 worked example of SURVEY Appendix C (s=0.5, M=1/1, q_bit=4,
 * delta=0, seed=1) and (2) the reference fixture random_tensor(32, 32, seed=7) (generated
 * on the device by sif_fixture_tensor, tensor.py:90-111; s=0.9, M=2/2, q_bit=8,
 * delta=0.01, seed=5 -- the CLI pipeline case of Appendix C), one sif_encode_batched call
 * per config, then decodes both payloads in ONE batched call with the device-side length
 * handoff (in_len_dev = the encoder's d_out_len), and prints
 *   payload <i> <hex>      and      decoded <i> <hex of the fp32 bits>
 * for tests/test_c_abi.py to compare with the reference's golden bytes.  Exit code != 0 on
 * any ABI or per-IF error. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "sif.h"

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));   \
      return 2;                                                                    \
    }                                                                              \
  } while (0)
#define ST(x)                                                                      \
  do {                                                                             \
    int s_ = (x);                                                                  \
    if (s_ != SIF_OK) {                                                            \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, sif_status_string(s_));    \
      return 3;                                                                    \
    }                                                                              \
  } while (0)

static void hexdump(const char* tag, int i, const unsigned char* p, size_t n) {
  printf("%s %d ", tag, i);
  for (size_t k = 0; k < n; ++k) printf("%02x", p[k]);
  printf("\n");
}

int main(void) {
  const float x6[6] = {3.f, -1.f, 0.5f, -4.f, 2.f, 0.1f};
  sif_codec_cfg cfgs[2];
  memset(cfgs, 0, sizeof(cfgs));
  cfgs[0].s = 0.5; cfgs[0].lam = 0.0; cfgs[0].delta = 0.0; cfgs[0].m_plus = 1; cfgs[0].m_minus = 1;
  cfgs[0].q_bit = 4; cfgs[0].mode = SIF_MODE_ABQ; cfgs[0].fixed_q = NULL;
  cfgs[1].s = 0.9; cfgs[1].lam = 0.0; cfgs[1].delta = 0.01; cfgs[1].m_plus = 2; cfgs[1].m_minus = 2;
  cfgs[1].q_bit = 8; cfgs[1].mode = SIF_MODE_ABQ; cfgs[1].fixed_q = NULL;
  ST(sif_validate_cfg(&cfgs[0]));
  ST(sif_validate_cfg(&cfgs[1]));

  const uint32_t rows[2] = {1, 32}, cols[2] = {6, 32};
  const uint64_t seeds[2] = {1, 5};
  float* dx[2];
  unsigned char* dout[2];
  uint64_t cap[2];
  CK(cudaMalloc((void**)&dx[0], 6 * sizeof(float)));
  CK(cudaMemcpy(dx[0], x6, sizeof(x6), cudaMemcpyHostToDevice));
  CK(cudaMalloc((void**)&dx[1], 32 * 32 * sizeof(float)));
  ST(sif_fixture_tensor(dx[1], 32 * 32, 7, 0, NULL)); /* random_tensor(32, 32, seed=7) */
  sif_enc_desc ed[2];
  memset(ed, 0, sizeof(ed));
  for (int i = 0; i < 2; ++i) {
    cap[i] = sif_max_payload_bytes(rows[i], cols[i], &cfgs[i]);
    CK(cudaMalloc((void**)&dout[i], cap[i]));
    ed[i].x = dx[i]; ed[i].out = dout[i]; ed[i].out_cap = cap[i]; ed[i].seed = seeds[i];
    ed[i].rows = rows[i]; ed[i].cols = cols[i]; ed[i].dtype = SIF_DTYPE_F32;
  }
  uint64_t* d_len = NULL;
  int32_t* d_st = NULL;
  CK(cudaMalloc((void**)&d_len, 2 * sizeof(uint64_t)));
  CK(cudaMalloc((void**)&d_st, 2 * sizeof(int32_t)));
  for (int i = 0; i < 2; ++i) {
    sif_plan plan;
    ST(sif_enc_plan(&ed[i], 1, &cfgs[i], &plan)); /* host only: the workspace size */
    void* ws = NULL;
    CK(cudaMalloc(&ws, plan.ws_bytes));
    ST(sif_encode_batched(&ed[i], 1, &cfgs[i], ws, plan.ws_bytes, d_len + i, d_st + i, NULL));
    CK(cudaDeviceSynchronize());
    CK(cudaFree(ws));
  }

  /* decode: lengths handed over on the device (no host round trip between the calls) */
  float* dy[2];
  sif_dec_desc dd[2];
  memset(dd, 0, sizeof(dd));
  for (int i = 0; i < 2; ++i) {
    CK(cudaMalloc((void**)&dy[i], (size_t)rows[i] * cols[i] * sizeof(float)));
    dd[i].in = dout[i]; dd[i].in_len = cap[i]; dd[i].out = dy[i]; dd[i].rows = rows[i]; dd[i].cols = cols[i];
    dd[i].in_len_dev = d_len + i;
  }
  sif_plan dplan;
  ST(sif_dec_plan(dd, 2, &dplan));
  void* dws = NULL;
  CK(cudaMalloc(&dws, dplan.ws_bytes));
  int32_t* d_dst = NULL;
  CK(cudaMalloc((void**)&d_dst, 2 * sizeof(int32_t)));
  ST(sif_decode_batched(dd, 2, 0, dws, dplan.ws_bytes, d_dst, NULL));
  CK(cudaDeviceSynchronize());

  uint64_t len[2];
  int32_t st[2], dst[2];
  CK(cudaMemcpy(len, d_len, sizeof(len), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(st, d_st, sizeof(st), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(dst, d_dst, sizeof(dst), cudaMemcpyDeviceToHost));
  for (int i = 0; i < 2; ++i) {
    if (st[i] != SIF_OK || dst[i] != SIF_OK) {
      fprintf(stderr, "IF %d: encode %s, decode %s\n", i, sif_status_string(st[i]), sif_status_string(dst[i]));
      return 4;
    }
    unsigned char* hp = (unsigned char*)malloc(len[i]);
    CK(cudaMemcpy(hp, dout[i], len[i], cudaMemcpyDeviceToHost));
    hexdump("payload", i, hp, len[i]);
    free(hp);
    const size_t nb = (size_t)rows[i] * cols[i] * sizeof(float);
    unsigned char* hy = (unsigned char*)malloc(nb);
    CK(cudaMemcpy(hy, dy[i], nb, cudaMemcpyDeviceToHost));
    hexdump("decoded", i, hy, nb);
    free(hy);
  }
  printf("ok\n");
  return 0;
}
