// Probe of TMA im2col-mode semantics on sm_100a (development tool, not product code).
// Loads 128-pixel x 64-channel im2col boxes of an NHWC uint16 tensor whose values encode
// (pixel, channel), copies SMEM back, and compares with the im2col of the convolution
// under the assumed semantics:
//   instruction coords {c, w, h, n} = input position of output pixel p0's filter origin
//   (wo*s - pad_w, ho*s - pad_h), offsets {dw, dh} = filter tap; pixel i of the box is
//   output pixel p0 + i in flat (n, ho, wo) order; out-of-range input -> 0.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/im2col_probe tools/im2col_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void k_probe(const __grid_constant__ CUtensorMap tm, int c0, int w0, int h0, int n0, int dw, int dh,
                        uint16_t* out) {
  __shared__ __align__(1024) uint8_t buf[128 * 128];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(buf);
  for (int i = threadIdx.x; i < 128 * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(buf)[i] = 0xDEADBEEF;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(128 * 128));
    const uint16_t ow = (uint16_t)dw, oh = (uint16_t)dh;
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
        "%6}], [%2], {%7, %8};" ::"r"(d),
        "l"(&tm), "r"(b), "r"(c0), "r"(w0), "r"(h0), "r"(n0), "h"(ow), "h"(oh)
        : "memory");
    asm volatile(
        "{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(b)
        : "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(buf)[i];
}

typedef CUresult (*EncIm2col)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const int*, const int*, cuuint32_t, cuuint32_t, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int N = 3, H = 12, W = 10, C = 64;
  std::vector<uint16_t> x((size_t)N * H * W * C);
  for (size_t p = 0; p < (size_t)N * H * W; ++p)
    for (int c = 0; c < C; ++c) x[p * C + c] = (uint16_t)(p * 64 + c + 1);
  uint16_t *dx, *dout;
  CK(cudaMalloc(&dx, x.size() * 2));
  CK(cudaMalloc(&dout, 128 * 64 * 2));
  CK(cudaMemcpy(dx, x.data(), x.size() * 2, cudaMemcpyHostToDevice));
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fp, cudaEnableDefault, &q));
  EncIm2col enc = (EncIm2col)fp;
  struct Case { int k_h, k_w, s, pad_h, pad_w; int swz; };
  Case cases[] = {{3, 3, 1, 1, 1, 0}, {3, 3, 2, 1, 1, 0}, {1, 1, 2, 0, 0, 0}, {7, 7, 2, 3, 3, 0}, {3, 3, 1, 1, 0, 0},
                  {3, 3, 1, 1, 1, 1}, {3, 3, 2, 1, 1, 1}};
  int total_bad = 0;
  for (const Case& cs : cases) {
    const int Ho = (H + 2 * cs.pad_h - cs.k_h) / cs.s + 1, Wo = (W + 2 * cs.pad_w - cs.k_w) / cs.s + 1;
    const int M = N * Ho * Wo;
    for (int order = 0; order < 2; ++order) {
      const int lw = -cs.pad_w, lh = -cs.pad_h;
      const int uw = (Wo - 1) * cs.s - cs.pad_w - (W - 1), uh = (Ho - 1) * cs.s - cs.pad_h - (H - 1);
      int lower[2], upper[2];
      if (order == 0) { lower[0] = lw; lower[1] = lh; upper[0] = uw; upper[1] = uh; }
      else { lower[0] = lh; lower[1] = lw; upper[0] = uh; upper[1] = uw; }
      cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
      cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
      cuuint32_t es[4] = {1, (cuuint32_t)cs.s, (cuuint32_t)cs.s, 1};
      CUtensorMap tm;
      CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, dx, dims, strides, lower, upper, 64, 128, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, cs.swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("case k%dx%d s%d p%d,%d order %d: encode failed %d\n", cs.k_h, cs.k_w, cs.s, cs.pad_h, cs.pad_w, order, (int)r); continue; }
      int bad = 0, checked = 0;
      const int p0s[3] = {0, 37, M > 130 ? M - 130 : 1};
      for (int pi = 0; pi < 3; ++pi)
        for (int tr = 0; tr < cs.k_h; tr += (cs.k_h > 1 ? cs.k_h - 1 : 1))
          for (int ts = 0; ts < cs.k_w; ts += (cs.k_w > 1 ? 1 : 1)) {
            const int p0 = p0s[pi];
            const int n0 = p0 / (Ho * Wo), ho0 = (p0 / Wo) % Ho, wo0 = p0 % Wo;
            k_probe<<<1, 128>>>(tm, 0, wo0 * cs.s - cs.pad_w, ho0 * cs.s - cs.pad_h, n0, ts, tr, dout);
            CK(cudaDeviceSynchronize());
            std::vector<uint16_t> o(128 * 64);
            CK(cudaMemcpy(o.data(), dout, o.size() * 2, cudaMemcpyDeviceToHost));
            for (int i = 0; i < 128; ++i) {
              const int p = p0 + i;
              for (int c = 0; c < 64; ++c) {
                uint16_t e = 0;
                if (p < M) {
                  const int n = p / (Ho * Wo), ho = (p / Wo) % Ho, wo = p % Wo;
                  const int hi = ho * cs.s - cs.pad_h + tr, wi = wo * cs.s - cs.pad_w + ts;
                  if (hi >= 0 && hi < H && wi >= 0 && wi < W) e = x[(((size_t)n * H + hi) * W + wi) * C + c];
                } else {
                  e = 0xFFFF;   // beyond the last output pixel: do not care
                }
                const int chunk = c / 8, phys = cs.swz ? (chunk ^ (i & 7)) : chunk;
                const uint16_t g = o[i * 64 + phys * 8 + (c & 7)];
                if (e == 0xFFFF) continue;
                ++checked;
                if (g != e) {
                  if (bad < 4 && order == 0)
                    printf("  mismatch k%dx%d s%d p0=%d tap(%d,%d) row %d c %d: got %u (pix %d c %d) want %u\n", cs.k_h,
                           cs.k_w, cs.s, p0, tr, ts, i, c, g, g ? (g - 1) / 64 : -1, g ? (g - 1) % 64 : -1, e);
                  ++bad;
                }
              }
            }
          }
      printf("case k%dx%d s%d pad(%d,%d) swz%d corner-order %d: %d / %d mismatches\n", cs.k_h, cs.k_w, cs.s, cs.pad_h,
             cs.pad_w, cs.swz, order, bad, checked);
      if (order == 0) total_bad += bad;
    }
  }
  printf("TOTAL order-0 mismatches %d\n", total_bad);
  return 0;
}
