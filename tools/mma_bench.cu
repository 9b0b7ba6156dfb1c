// Microbenchmark: cycles per tcgen05.mma (M=128, K=16, bf16) for several N, issued
// back-to-back by one thread into one TMEM accumulator, operands in SMEM (no-swizzle
// K-major layout as in conv_tma.cu).  Also measures the warp-uniform issue variant.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_bench tools/mma_bench.cu
#include <cstdio>
#include <cstdint>
#include "../paper_2307_04963_b200/csrc/ptx.cuh"

using namespace dycl;

template <int N, bool UNIFORM>
__global__ void k_mma(int iters, long long* out) {
  __shared__ __align__(1024) uint8_t sA[128 * 16 * 2 * 2];   // 2 K chunks of 128 rows x 16 B
  __shared__ __align__(1024) uint8_t sB[256 * 16 * 2];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < (int)sizeof(sA) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sA)[i] = 0;
  for (int i = threadIdx.x; i < (int)sizeof(sB) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sB)[i] = 0;
  const uint32_t barA = ptx::smem_u32(&bar);
  if (threadIdx.x == 0) {
    ptx::mbar_init(barA, 1);
    ptx::fence_mbar_init();
  }
  if (threadIdx.x < 32) ptx::tmem_alloc(ptx::smem_u32(&slot), 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t idesc = ptx::make_idesc_bf16(128, N);
  const uint64_t ad = ptx::make_smem_desc(ptx::smem_u32(sA), 0, 128 * 16, 128);
  const uint64_t bd = ptx::make_smem_desc(ptx::smem_u32(sB), 0, N * 16, 128);
  long long t0 = 0, t1 = 0;
  if (threadIdx.x < 32) {
    if (UNIFORM) {
      t0 = clock64();
      for (int i = 0; i < iters; ++i) {
        asm volatile(
            "{\n\t.reg .pred p, e;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"(i)
            : "memory");
      }
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(barA)
          : "memory");
      ptx::mbar_wait(barA, 0);
      t1 = clock64();
    } else if (threadIdx.x == 0) {
      t0 = clock64();
      for (int i = 0; i < iters; ++i) ptx::mma_bf16_ss(tmem, ad, bd, idesc, i != 0);
      ptx::mma_commit(barA);
      ptx::mbar_wait(barA, 0);
      t1 = clock64();
    }
  }
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

template <int N, bool U>
void run(int blocks) {
  long long* d;
  cudaMalloc(&d, blocks * sizeof(long long));
  const int iters = 4096;
  k_mma<N, U><<<blocks, 128>>>(iters, d);
  k_mma<N, U><<<blocks, 128>>>(iters, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_mma<N, U><<<blocks, 128>>>(iters, d);
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h;
  cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double flops = 2.0 * 128 * N * 16 * iters * blocks;
  printf("N=%3d %s blocks=%3d: %6.1f cycles/MMA (clock64), %7.1f TFLOP/s  (%s)\n", N, U ? "uniform " : "lane0   ",
         blocks, (double)h / iters, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<16, false>(148); run<16, true>(148);
  run<32, false>(148); run<32, true>(148);
  run<64, false>(148); run<64, true>(148);
  run<128, false>(148); run<128, true>(148);
  run<256, false>(148); run<256, true>(148);
  run<16, true>(1);
  run<256, true>(1);
  return 0;
}
