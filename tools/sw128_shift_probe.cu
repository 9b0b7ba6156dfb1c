// Probe (development tool, not product code): can a tcgen05 K-major SWIZZLE_128B operand start
// at an arbitrary 128-byte row inside the 1024-byte swizzle atom?  The A tile is written with
// the address-based 128B swizzle (chunk j of row r at base + r*128 + ((j ^ (r & 7)) << 4), the
// image TMA produces), then MMAs 128 x 64 x 64 read rows v .. v+127 through a descriptor whose
// start address is base + 128 v (+ 32 B per K step), with the descriptor's base-offset field
// either 0 or (v & 7).  Each variant is compared with the exact integer product.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -I paper_2307_04963_b200/csrc -o /tmp/sw128_probe tools/sw128_shift_probe.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#include "ptx.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

constexpr int AROWS = 160, NB = 64, VMAX = 24;

__global__ void k_probe(const uint16_t* A, const uint16_t* B, float* out) {
  __shared__ __align__(1024) uint8_t sA[AROWS * 128];
  __shared__ __align__(1024) uint8_t sB[NB * 128];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < AROWS * 8; i += blockDim.x) {
    const int r = i / 8, j = i % 8;
    *reinterpret_cast<uint4*>(sA + r * 128 + ((j ^ (r & 7)) << 4)) = *reinterpret_cast<const uint4*>(A + r * 64 + j * 8);
  }
  for (int i = threadIdx.x; i < NB * 8; i += blockDim.x) {
    const int r = i / 8, j = i % 8;
    *reinterpret_cast<uint4*>(sB + r * 128 + ((j ^ (r & 7)) << 4)) = *reinterpret_cast<const uint4*>(B + r * 64 + j * 8);
  }
  dycl::ptx::fence_proxy_async_smem();
  const uint32_t b = dycl::ptx::smem_u32(&bar);
  if (threadIdx.x == 0) {
    dycl::ptx::mbar_init(b, 1);
    dycl::ptx::fence_mbar_init();
  }
  if (warp == 0) dycl::ptx::tmem_alloc(dycl::ptx::smem_u32(&slot), 64);
  dycl::ptx::tc_fence_before();
  __syncthreads();
  dycl::ptx::tc_fence_after();
  const uint32_t tmem = slot;
  constexpr uint32_t IDESC = dycl::ptx::make_idesc_bf16(128, NB);
  uint32_t ph = 0;
  for (int v = 0; v < VMAX; ++v)
    for (int mode = 0; mode < 2; ++mode) {
      if (warp == 0) {
        for (int j = 0; j < 4; ++j) {
          uint64_t ad = dycl::ptx::make_smem_desc_sw128(dycl::ptx::smem_u32(sA) + 128 * v + 32 * j);
          if (mode == 1) ad |= (uint64_t)(v & 7) << 49;
          const uint64_t bd = dycl::ptx::make_smem_desc_sw128(dycl::ptx::smem_u32(sB) + 32 * j);
          dycl::ptx::mma_bf16_ss_elect(tmem, ad, bd, IDESC, j != 0);
        }
        dycl::ptx::mma_commit_elect(b);
      }
      dycl::ptx::mbar_wait(b, ph);
      ph ^= 1;
      dycl::ptx::tc_fence_after();
      for (int c0 = 0; c0 < NB; c0 += 16) {
        uint32_t t[16];
        dycl::ptx::tmem_ld_32x32b_x16(tmem + ((uint32_t)(warp * 32) << 16) + c0, t);
        dycl::ptx::tmem_ld_wait();
        for (int q = 0; q < 16; ++q)
          out[(((size_t)v * 2 + mode) * 128 + warp * 32 + lane) * NB + c0 + q] = __uint_as_float(t[q]);
      }
      dycl::ptx::tc_fence_before();
      __syncthreads();
      dycl::ptx::tc_fence_after();
    }
  __syncthreads();
  if (warp == 0) dycl::ptx::tmem_dealloc(tmem, 64);
}

static uint16_t bf(float f) {
  __nv_bfloat16 h = __float2bfloat16(f);
  return *reinterpret_cast<uint16_t*>(&h);
}

int main() {
  std::vector<float> a(AROWS * 64), bm(NB * 64);
  std::vector<uint16_t> ah(a.size()), bh(bm.size());
  srand(7);
  for (size_t i = 0; i < a.size(); ++i) { a[i] = (float)(rand() % 7 - 3); ah[i] = bf(a[i]); }
  for (size_t i = 0; i < bm.size(); ++i) { bm[i] = (float)(rand() % 5 - 2); bh[i] = bf(bm[i]); }
  uint16_t *dA, *dB;
  float* dO;
  const size_t on = (size_t)VMAX * 2 * 128 * NB;
  CK(cudaMalloc(&dA, ah.size() * 2));
  CK(cudaMalloc(&dB, bh.size() * 2));
  CK(cudaMalloc(&dO, on * 4));
  CK(cudaMemcpy(dA, ah.data(), ah.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, bh.data(), bh.size() * 2, cudaMemcpyHostToDevice));
  k_probe<<<1, 128>>>(dA, dB, dO);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> o(on);
  CK(cudaMemcpy(o.data(), dO, on * 4, cudaMemcpyDeviceToHost));
  for (int mode = 0; mode < 2; ++mode) {
    printf("base_offset %s:", mode ? "= v & 7" : "= 0    ");
    for (int v = 0; v < VMAX; ++v) {
      int bad = 0;
      for (int i = 0; i < 128; ++i)
        for (int n = 0; n < NB; ++n) {
          float e = 0;
          for (int k = 0; k < 64; ++k) e += a[(v + i) * 64 + k] * bm[n * 64 + k];
          bad += o[(((size_t)v * 2 + mode) * 128 + i) * NB + n] != e;
        }
      printf(" v%d:%s", v, bad ? "BAD" : "ok");
    }
    printf("\n");
  }
  return 0;
}
