// Fused conv epilogue shared by the tensor-core conv kernels:
//   y = act(acc + bias [+ shortcut])  -> bf16 operand copy (channel-planar layout)
//                                      (+ fp32 residual-stream copy, NHWC)
// Layouts:
//   bf16 activations: channel-planar "NC8HW8"  [n][C/8][H][W][8]  (16-byte pixel chunks;
//                     a TMA box row is then a whole image row of one 8-channel plane)
//   fp32 stream:      NHWC                     [n][H][W][C]
//   (ConvArgs.nhwc: bf16 activations NHWC as well -- the config-5 layout)
#pragma once
#include <cuda_bf16.h>

#include "kernels.h"

namespace dycl {

__device__ __forceinline__ uint32_t pack_bf16x2_rn(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// f[16]: fp32 accumulators of output channels o0..o0+15 of pixel (n, ho, wo).
// bias_s: the bias staged in shared memory (or nullptr -> read a.bias);
// res_s : this pixel's 16 fp32 identity-shortcut values already in shared memory
//         (prefetched by the TMA producer), or nullptr -> read from global.
__device__ __forceinline__ void conv_finish16(const ConvArgs& a, int n, int ho, int wo, int o0, float (&f)[16],
                                              const float* bias_s = nullptr, const float* res_s = nullptr) {
  const size_t HWo = (size_t)a.Ho * a.Wo;
  const size_t pix = (size_t)ho * a.Wo + wo;
  if (bias_s) {
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      const float4 q = *reinterpret_cast<const float4*>(bias_s + o0 + j);
      f[j] += q.x; f[j + 1] += q.y; f[j + 2] += q.z; f[j + 3] += q.w;
    }
  } else {
    // four broadcast 16-byte loads (o0 is a multiple of 16) instead of sixteen scalar ones
    const float4* b4 = reinterpret_cast<const float4*>(a.bias + o0);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 q = __ldg(b4 + j);
      f[4 * j] += q.x; f[4 * j + 1] += q.y; f[4 * j + 2] += q.z; f[4 * j + 3] += q.w;
    }
  }
  if (a.res_mode == 1 && res_s) {
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      const float4 q = *reinterpret_cast<const float4*>(res_s + j);
      f[j] += q.x; f[j + 1] += q.y; f[j + 2] += q.z; f[j + 3] += q.w;
    }
  } else if (a.res_mode == 1) {
    if (a.res32) {
      const float4* rp = reinterpret_cast<const float4*>(a.res32 + ((size_t)n * HWo + pix) * a.Cout + o0);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float4 q = __ldg(rp + j);
        f[4 * j] += q.x; f[4 * j + 1] += q.y; f[4 * j + 2] += q.z; f[4 * j + 3] += q.w;
      }
    } else {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint4 r = __ldg(reinterpret_cast<const uint4*>(
            a.nhwc ? a.res + ((size_t)n * HWo + pix) * a.Cout + o0 + 8 * h
                   : a.res + (size_t)n * a.Cout * HWo + (size_t)((o0 >> 3) + h) * HWo * 8 + pix * 8));
        const uint32_t u[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          f[8 * h + 2 * j] += __uint_as_float(u[j] << 16);
          f[8 * h + 2 * j + 1] += __uint_as_float(u[j] & 0xFFFF0000u);
        }
      }
    }
  } else if (a.res_mode == 2 && a.r_pad_lo % 4 == 0 && a.rC % 4 == 0 && !a.res_nhwc) {
    // option A, vectorised: r_pad_lo and rC are multiples of 4, so each 4-channel group is
    // entirely inside or outside [0, rC): one 16-byte (fp32) / 8-byte (bf16) load per group
    const size_t rHW = (size_t)a.rH * a.rW;
    const size_t rpix = (size_t)(2 * ho) * a.rW + 2 * wo;
#pragma unroll
    for (int g4 = 0; g4 < 4; ++g4) {
      const int ci = o0 + 4 * g4 - a.r_pad_lo;
      if (ci < 0 || ci + 4 > a.rC) continue;
      float4 q;
      if (a.res32) {
        q = __ldg(reinterpret_cast<const float4*>(a.res32 + ((size_t)n * rHW + rpix) * a.rC + ci));
      } else {
        const uint2 u = __ldg(reinterpret_cast<const uint2*>(a.res + (size_t)n * a.rC * rHW + (size_t)(ci >> 3) * rHW * 8 +
                                                             rpix * 8 + (ci & 7)));
        q = make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u), __uint_as_float(u.y << 16),
                        __uint_as_float(u.y & 0xFFFF0000u));
      }
      f[4 * g4] += q.x; f[4 * g4 + 1] += q.y; f[4 * g4 + 2] += q.z; f[4 * g4 + 3] += q.w;
    }
  } else if (a.res_mode == 2) {
    // option A: shortcut = input pixel (2ho, 2wo), channel o - r_pad_lo (zero outside [0, rC))
    const size_t rHW = (size_t)a.rH * a.rW;
    const size_t rpix = (size_t)(2 * ho) * a.rW + 2 * wo;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int ci = o0 + j - a.r_pad_lo;
      if (ci >= 0 && ci < a.rC) {
        f[j] += a.res32 ? __ldg(a.res32 + ((size_t)n * rHW + rpix) * a.rC + ci)
                        : __uint_as_float((uint32_t)a.res[(size_t)n * a.rC * rHW + (size_t)(ci >> 3) * rHW * 8 +
                                                           rpix * 8 + (ci & 7)] << 16);
      }
    }
  }
  if (a.relu) {
#pragma unroll
    for (int j = 0; j < 16; ++j) f[j] = fmaxf(f[j], 0.0f);
  }
  if (a.split && a.y) {                 // dense split pair: hi at [row][o], lo at [row][Cout + o]
    uint16_t* yr = a.y + (size_t)n * 2 * a.Cout + o0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint4 hi, lo;
      uint32_t* hp = &hi.x;
      uint32_t* lp = &lo.x;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float v0 = f[8 * h + 2 * j], v1 = f[8 * h + 2 * j + 1];
        hp[j] = pack_bf16x2_rn(v0, v1);
        lp[j] = pack_bf16x2_rn(v0 - __uint_as_float(hp[j] << 16), v1 - __uint_as_float(hp[j] & 0xFFFF0000u));
      }
      *reinterpret_cast<uint4*>(yr + 8 * h) = hi;
      *reinterpret_cast<uint4*>(yr + a.Cout + 8 * h) = lo;
    }
  }
#pragma unroll
  for (int h = 0; h < 2 && a.y && !a.split; ++h) {
    uint4 o;
    o.x = pack_bf16x2_rn(f[8 * h + 0], f[8 * h + 1]);
    o.y = pack_bf16x2_rn(f[8 * h + 2], f[8 * h + 3]);
    o.z = pack_bf16x2_rn(f[8 * h + 4], f[8 * h + 5]);
    o.w = pack_bf16x2_rn(f[8 * h + 6], f[8 * h + 7]);
    *reinterpret_cast<uint4*>(a.nhwc ? a.y + ((size_t)n * HWo + pix) * a.Cout + o0 + 8 * h
                                     : a.y + (size_t)n * a.Cout * HWo + (size_t)((o0 >> 3) + h) * HWo * 8 + pix * 8) = o;
  }
  if (a.y32) {
    const size_t ld = a.y32_ld ? (size_t)a.y32_ld : (size_t)a.Cout;
    const int nv = a.y32_n ? a.y32_n : a.Cout;
    float4* yq = reinterpret_cast<float4*>(a.y32 + ((size_t)n * HWo + pix) * ld + o0);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (o0 + 4 * j < nv) yq[j] = make_float4(f[4 * j], f[4 * j + 1], f[4 * j + 2], f[4 * j + 3]);
  }
}

}  // namespace dycl
