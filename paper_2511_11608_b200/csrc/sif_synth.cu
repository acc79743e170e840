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

namespace sif {

// ---------------------------------------------------------------------------------------
// Fixture tensors of the reference (tensor.py:90-111, rng.py:30-52) generated on the device.
// The splitmix64 stream is counter based: draw n is mix(seed + (n+1)*golden), so element i
// of a uniform tensor is draw i and gaussian pair p uses draws 2p and 2p+1.
//   uniform:  f32(-1 + 2 * (f64(u) / 2^64))                         (rng.py:41-45)
//   gaussian: u1 = f64(u_2p + 1) / 2^64, u2 = f64(u_2p+1) / 2^64,
//             r = sqrt(-2 log u1); (r cos(2 pi u2), r sin(2 pi u2))  (rng.py:47-52)
// Every fp64 step is the same IEEE operation the reference performs (int -> double is
// round-to-nearest in both; / 2^64 is exact), so uniform tensors are bit-identical.  The
// gaussian path calls CUDA's log/sqrt/sin/cos: sqrt is correctly rounded, log/sin/cos are
// within 1-2 ulp of glibc's, which changes the fp32 result only when the fp64 value lies
// within a few fp64 ulp of an fp32 rounding boundary.
__global__ void sif_fixture_kernel(float* x, uint64_t n, uint64_t seed, uint32_t dist) {
  const double two64 = 18446744073709551616.0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    if (dist == 0) {
      const double unit = __ddiv_rn(__ull2double_rn(splitmix(seed, i)), two64);
      x[i] = __double2float_rn(__dadd_rn(-1.0, __dmul_rn(2.0, unit)));
    } else {
      const uint64_t p = i >> 1;
      const uint64_t a = splitmix(seed, 2 * p), b = splitmix(seed, 2 * p + 1);
      // (a + 1) as a Python int may be 2^64: convert a, then add one exactly in the
      // rounding of the conversion (a + 1 < 2^64 unless a = 2^64 - 1)
      const double a1 = a == 0xFFFFFFFFFFFFFFFFull ? two64 : __ull2double_rn(a + 1ull);
      const double u1 = __ddiv_rn(a1, two64), u2 = __ddiv_rn(__ull2double_rn(b), two64);
      const double r = __dsqrt_rn(__dmul_rn(-2.0, log(u1)));
      const double ang = __dmul_rn(__dmul_rn(2.0, 3.141592653589793), u2);
      const double v = (i & 1) ? __dmul_rn(r, sin(ang)) : __dmul_rn(r, cos(ang));
      x[i] = __double2float_rn(v);
    }
  }
}

// Count of non-finite fp32 elements (tensor.py:35-36 / :84-85); *count must be zeroed.
__global__ void sif_nonfinite_kernel(const uint32_t* x, uint64_t n, unsigned long long* count) {
  uint32_t c = 0;
  const uint64_t n4 = n / 4;
  const uint4* x4 = reinterpret_cast<const uint4*>(x);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldg(x4 + i);
    c += ((v.x & 0x7F800000u) == 0x7F800000u) + ((v.y & 0x7F800000u) == 0x7F800000u) +
         ((v.z & 0x7F800000u) == 0x7F800000u) + ((v.w & 0x7F800000u) == 0x7F800000u);
  }
  for (uint64_t i = 4 * n4 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    c += (x[i] & 0x7F800000u) == 0x7F800000u;
  c = __reduce_add_sync(0xFFFFFFFFu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, (unsigned long long)c);
}

}  // namespace sif
