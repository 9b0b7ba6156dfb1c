// Implicit-GEMM convolution / dense layer on 5th-generation tensor cores (sm_100a).
//
// Row-sample activations (NHWC bf16) x weights [Cout][k*k*C] -> bf16 NHWC output,
// with the bias / shortcut / ReLU / bf16-rounding epilogue fused.
//
//   D[m, o] = sum_k A[m, k] * B[o, k]
//   m = (n, ho, wo) output pixel,  k = (r, s, c) tap x input channel,  o = out channel
//   A[m, k] = x[n][ho*stride - pad + r][wo*stride - pad + s][c]   (0 outside the image)
//
// Persistent, warp-specialised CTA (one per SM):
//   warps 0-3  epilogue: tcgen05.ld TMEM -> regs -> conv_finish16 (bias, shortcut,
//              ReLU, bf16 channel-planar + fp32 NHWC stores; epilogue.cuh)
//   warps 4-11 producers: im2col gather of A and the B tile with 16-byte
//              cp.async (zero-fill implements the padding) into a STAGES-deep ring
//              laid out in the UMMA 128B-swizzle K-major canonical layout; the
//              per-chunk tap geometry (r, s, c) is row-independent and read from a
//              shared-memory table built once per CTA (no divisions in the loop)
//   warp  12   TMEM allocator + MMA issuer: one lane issues tcgen05.mma
//              (M=128, N=BN, K=16) and tcgen05.commit to free ring slots and to
//              hand a finished accumulator to the epilogue
// Two TMEM accumulators (2*BN columns) let the epilogue of tile i overlap the
// MMAs of tile i+1.  The live-row count is read from device memory, so the same
// launch serves every batch the host module produces without a host round trip.
#include <cuda_bf16.h>

#include "epilogue.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace dycl {
namespace {

constexpr int BM = 128;
constexpr int BK = 64;          // bf16 elements per K block = one 128-byte swizzle row
constexpr int NUM_PRODUCERS = 256;   // 8 warps: two threads per A row, 4 chunks each
constexpr int NUM_THREADS = 128 + NUM_PRODUCERS + 32;
constexpr int MMA_WARP = (128 + NUM_PRODUCERS) / 32;
constexpr int MAX_KCH = 1024;        // K chunks (8 elements) covered by the tap table (K <= 8192)

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (196608 / STAGE_BYTES) > 8 ? 8 : (196608 / STAGE_BYTES);
  static constexpr int TMEM_COLS = (2 * BN) <= 32 ? 32 : (2 * BN) <= 64 ? 64 : (2 * BN) <= 128 ? 128
                                   : (2 * BN) <= 256 ? 256 : 512;
  static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + 256 + MAX_KCH * 8;
  // Producer lag: each producer thread keeps LAG cp.async groups (ring fills) in
  // flight before it arrives on the oldest fill's full barrier.  LAG <= STAGES-1
  // is deadlock-free: before issuing fill f+1 the producer waits for the MMA to
  // release fill f+1-STAGES, and every fill <= f-LAG has already been arrived.
  static constexpr int LAG = STAGES - 1;
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA M=128 needs N%16==0, 16<=N<=256");
};


template <int BN>
__global__ void __launch_bounds__(NUM_THREADS, 1) k_conv_tc(const ConvArgs a) {
  using C = Cfg<BN>;
  constexpr int S = C::STAGES;
  constexpr int LAG = C::LAG;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * C::A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + S * C::B_BYTES);
  const uint32_t full0 = ptx::smem_u32(bars);
  const uint32_t empty0 = full0 + 8 * S;
  const uint32_t tfull0 = empty0 + 8 * S;
  const uint32_t tempty0 = tfull0 + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 4);
  int2* tap_tab = reinterpret_cast<int2*>(reinterpret_cast<uint8_t*>(bars) + 256);   // [Kp/8]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  const int n_live = a.n_live ? *a.n_live : a.n_static;
  const int HoWo = a.Ho * a.Wo;
  const long long M = (long long)n_live * HoWo;
  const int m_tiles = (int)((M + BM - 1) / BM);
  const int n_tiles = a.Cout / BN;
  const int num_tiles = m_tiles * n_tiles;
  const int ksteps = (a.K + 15) >> 4;
  const int kblocks = (ksteps + 3) >> 2;

  // tap table: chunk j covers k = 8j..8j+7 = tap (r, s), channels c..c+7 = plane c/8
  // of the channel-planar input [n][C/8][H][W][8].
  //   .x = element offset (c/8)*H*W*8 + (r*W + s)*8 from the window origin,
  //   .y = (r << 16) | s;  .y = -1 marks chunks beyond K (zero-filled).
  for (int j = threadIdx.x; j < a.Kp / 8 && j < MAX_KCH; j += blockDim.x) {
    const int k = j * 8;
    if (k < a.K) {
      const int tap = k / a.C, c = k - (k / a.C) * a.C;
      const int r = tap / a.ksz, s2 = tap - (tap / a.ksz) * a.ksz;
      tap_tab[j] = make_int2((c >> 3) * a.H * a.W * 8 + (r * a.W + s2) * 8, (r << 16) | s2);
    } else {
      tap_tab[j] = make_int2(0, -1);
    }
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      ptx::mbar_init(full0 + 8 * i, NUM_PRODUCERS);
      ptx::mbar_init(empty0 + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(tfull0 + 8 * i, 1);
      ptx::mbar_init(tempty0 + 8 * i, 128);
    }
    ptx::fence_mbar_init();
  }
  if (warp == MMA_WARP) ptx::tmem_alloc(ptx::smem_u32(tmem_slot), C::TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp >= 4 && warp < MMA_WARP) {
    // ------------------------------------------------------------ producers
    const int t = threadIdx.x - 128;
    const int row = t & 127;                 // A row of the tile this thread fills
    const int qh = (t >> 7) * 4;             // its chunks: qh .. qh+3 of every K block
    const uint32_t a_row_off = (uint32_t)((row >> 3) * 1024 + (row & 7) * 128);
    const int sw = row & 7;
    int stage = 0;
    uint32_t phase = 0;
    int issued = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int m_tile = tile / n_tiles;
      const int n_tile = tile - m_tile * n_tiles;
      const long long m = (long long)m_tile * BM + row;
      const bool row_ok = m < M;
      int n = 0, ho = 0, wo = 0;
      if (row_ok) {
        n = (int)(m / HoWo);
        const int p = (int)(m - (long long)n * HoWo);
        ho = p / a.Wo;
        wo = p - ho * a.Wo;
      }
      const int hi0 = ho * a.stride - a.pad;
      const int wi0 = wo * a.stride - a.pad;
      // window origin (may point before the sample for padded rows; only used when in bounds)
      const long long base = (long long)n * a.H * a.W * a.C + ((long long)hi0 * a.W + wi0) * 8;
      const uint16_t* wt = a.w + (size_t)n_tile * BN * a.Kp;
      for (int kb = 0; kb < kblocks; ++kb) {
        ptx::mbar_wait(empty0 + 8 * stage, phase ^ 1);
        const int kused = min(BK, ksteps * 16 - kb * BK);   // K elements the MMAs read in this block
        const uint32_t sa = ptx::smem_u32(sA + stage * C::A_BYTES) + a_row_off;
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          const int q = qh + qq;
          if (q * 8 < kused) {
            const int2 tb = tap_tab[kb * 8 + q];
            const int r = tb.y >> 16, s2 = tb.y & 0xFFFF;
            const void* src = a.x;
            uint32_t bytes = 0;
            if (row_ok && tb.y >= 0 && (unsigned)(hi0 + r) < (unsigned)a.H && (unsigned)(wi0 + s2) < (unsigned)a.W) {
              src = a.x + base + tb.x;
              bytes = 16;
            }
            ptx::cp_async_16_ca(sa + (uint32_t)((q ^ sw) << 4), src, bytes);
          }
        }
        const uint32_t sb = ptx::smem_u32(sB + stage * C::B_BYTES);
        for (int i = t; i < BN * 8; i += NUM_PRODUCERS) {
          const int nrow = i % BN;
          const int q = i / BN;
          if (q * 8 < kused) {
            const uint16_t* src = wt + (size_t)nrow * a.Kp + kb * BK + q * 8;
            ptx::cp_async_16_cg(sb + (uint32_t)((nrow >> 3) * 1024 + (nrow & 7) * 128 + ((q ^ (nrow & 7)) << 4)),
                                src, 16);
          }
        }
        ptx::cp_async_commit();
        ++issued;
        if (issued > LAG) {
          ptx::cp_async_wait<LAG>();
          ptx::fence_proxy_async_smem();
          ptx::mbar_arrive(full0 + 8 * ((stage - LAG + S) % S));
        }
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    ptx::cp_async_wait<0>();
    ptx::fence_proxy_async_smem();
    const int pend = issued < LAG ? issued : LAG;
    for (int j = pend; j >= 1; --j) ptx::mbar_arrive(full0 + 8 * ((stage - j + S) % S));
  } else if (warp == MMA_WARP) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t IDESC = ptx::make_idesc_bf16(BM, BN);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      ptx::mbar_wait(tempty0 + 8 * acc, acc_phase ^ 1);
      ptx::tc_fence_after();
      const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
      for (int kb = 0; kb < kblocks; ++kb) {
        ptx::mbar_wait(full0 + 8 * stage, phase);
        ptx::tc_fence_after();
        if (lane == 0) {
          const int nsteps = min(4, ksteps - kb * 4);
          const uint32_t sa = ptx::smem_u32(sA + stage * C::A_BYTES);
          const uint32_t sb = ptx::smem_u32(sB + stage * C::B_BYTES);
          for (int j = 0; j < nsteps; ++j) {
            ptx::mma_bf16_ss(d_tmem, ptx::make_smem_desc_sw128(sa + 32 * j), ptx::make_smem_desc_sw128(sb + 32 * j),
                             IDESC, (kb | j) != 0);
          }
          ptx::mma_commit(empty0 + 8 * stage);
        }
        __syncwarp();
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (lane == 0) ptx::mma_commit(tfull0 + 8 * acc);
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int row = warp * 32 + lane;
    int it = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int m_tile = tile / n_tiles;
      const int n_tile = tile - m_tile * n_tiles;
      const long long m = (long long)m_tile * BM + row;
      const bool ok = m < M;
      ptx::mbar_wait(tfull0 + 8 * acc, acc_phase);
      ptx::tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(warp * 32) << 16) + (uint32_t)(acc * BN);
      int n = 0, ho = 0, wo = 0;
      if (ok) {
        n = (int)(m / HoWo);
        const int p = (int)(m - (long long)n * HoWo);
        ho = p / a.Wo;
        wo = p - ho * a.Wo;
      }
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t v[16];
        ptx::tmem_ld_32x32b_x16(taddr + (uint32_t)c0, v);
        ptx::tmem_ld_wait();
        if (ok) {
          float f[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) f[j] = __uint_as_float(v[j]);
          conv_finish16(a, n, ho, wo, n_tile * BN + c0, f);
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(tempty0 + 8 * acc);
    }
  }

  __syncthreads();
  if (warp == MMA_WARP) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

template <int BN>
cudaError_t launch_bn(const ConvArgs& a, int max_rows, int num_sms, cudaStream_t stream) {
  using C = Cfg<BN>;
  if (cudaError_t e = ensure_smem(k_conv_tc<BN>, C::SMEM_BYTES)) return e;
  const long long max_m = (long long)max_rows * a.Ho * a.Wo;
  const long long tiles = ((max_m + BM - 1) / BM) * (a.Cout / BN);
  int grid = (int)(tiles < num_sms ? tiles : num_sms);
  if (grid < 1) grid = 1;
  k_conv_tc<BN><<<grid, NUM_THREADS, C::SMEM_BYTES, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_conv_tc(const ConvArgs& a, int max_rows, int num_sms, cudaStream_t stream) {
  if (a.Kp / 8 > MAX_KCH || a.C % 8 != 0) return cudaErrorInvalidValue;
  // N tile: the whole Cout when it fits one UMMA (<= 256), else 256 / 128 tiles.
  if (a.Cout <= 256) {
    switch (a.Cout) {
      case 16: return launch_bn<16>(a, max_rows, num_sms, stream);
      case 32: return launch_bn<32>(a, max_rows, num_sms, stream);
      case 48: return launch_bn<48>(a, max_rows, num_sms, stream);
      case 64: return launch_bn<64>(a, max_rows, num_sms, stream);
      case 96: return launch_bn<96>(a, max_rows, num_sms, stream);
      case 128: return launch_bn<128>(a, max_rows, num_sms, stream);
      case 192: return launch_bn<192>(a, max_rows, num_sms, stream);
      case 256: return launch_bn<256>(a, max_rows, num_sms, stream);
      default: break;
    }
  }
  if (a.Cout % 256 == 0) return launch_bn<256>(a, max_rows, num_sms, stream);
  if (a.Cout % 128 == 0) return launch_bn<128>(a, max_rows, num_sms, stream);
  if (a.Cout % 64 == 0) return launch_bn<64>(a, max_rows, num_sms, stream);
  if (a.Cout % 16 == 0) return launch_bn<16>(a, max_rows, num_sms, stream);
  return cudaErrorInvalidValue;
}

// Lazy-loading anchor: a kernel of this translation unit's module (preload_kernels, hostmod.cu).
__global__ void k_tu_anchor_conv_tc() {}
const void* tu_anchor_conv_tc() { return reinterpret_cast<const void*>(&k_tu_anchor_conv_tc); }

}  // namespace dycl
