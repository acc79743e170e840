// sif_synth.cu -- integer-exact synthetic IF generator on the device.
// Bit-identical to oracle/synth.py; used by bench.py and the GPU tests to create inputs
// directly in HBM.  Not part of the codec path.
#include <stdint.h>

#include "sif_common.cuh"

namespace sif {

__device__ __forceinline__ float synth_gauss(uint64_t sid, uint64_t i) {
  const uint64_t u = splitmix(sid, i);
  int64_t z = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) z += (int64_t)((u >> (16 * j)) & 0xFFFFull);
  z -= 131070;
  return __fmul_rn((float)z, 3.0517578125e-05f);  // 2^-15, exact
}

__device__ __forceinline__ uint32_t bf16_rne_bits(float f) {
  const uint32_t b = __float_as_uint(f);
  return ((b + 0x7FFFu + ((b >> 16) & 1u)) & 0xFFFF0000u);
}

__global__ void sif_synth_kernel(void* x, uint32_t rows, uint32_t cols, uint32_t dtype, uint32_t kind,
                                 uint64_t sid) {
  const uint64_t T = (uint64_t)rows * cols;
  uint32_t outlier[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) outlier[j] = (uint32_t)(splitmix(sid ^ 0xA5ull, (uint64_t)j) % (uint64_t)cols);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < T; i += (uint64_t)gridDim.x * blockDim.x) {
    const float g = synth_gauss(sid, i);
    uint32_t bits;
    if (kind == 0) {  // ResNet ReLU IF: max(0, g + b_c), b_c = -(c mod 4)/4
      const uint32_t c = (uint32_t)(i / cols);
      const float bias = -(float)(c % 4u) * 0.25f;
      const float v = __fadd_rn(g, bias);
      bits = __float_as_uint(v > 0.0f ? v : 0.0f);
    } else {  // LLM hidden state: bf16_rne(g * a_h)
      const uint32_t h = (uint32_t)(i % cols);
      float a = 1.0f;
#pragma unroll
      for (int j = 0; j < 8; ++j) if (outlier[j] == h) a = 32.0f;
      bits = bf16_rne_bits(__fmul_rn(g, a));
    }
    if (dtype == SIF_DTYPE_F32) reinterpret_cast<uint32_t*>(x)[i] = bits;
    else reinterpret_cast<unsigned short*>(x)[i] = (unsigned short)(bits >> 16);
  }
}

}  // namespace sif
