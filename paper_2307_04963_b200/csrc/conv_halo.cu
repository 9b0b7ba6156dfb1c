// KxK / stride-1 NHWC convolution with a TMA halo tile and shifted UMMA descriptors
// (the ResNet-50 stage-1 bottleneck conv2, 3x3 56x56x64 -> 64, the stem in
// its 4x4 space-to-depth form, 3x3 over 56x56x64 -> 256, and the opt-in 2x2 form of the stem,
// 4x4 over 112x112x16 -> 64).
//
// The im2col GEMM (conv_gemm.cu) loads one TMA im2col box per tap: 9 x 16 KB of A per 128-row
// tile, and on the 64-channel 3x3 layers that operand feed (not the tensor core) bounds it
// (ncu: tensor pipe 26 %, producer / full-barrier waits on top; profiles/r02_ncu_conv_gemm_cfg5.txt).
// Here a tile is R whole output rows of one sample.  Its input with the 1-pixel halo -- rows
// y0-1 .. y0+R, columns -1 .. W -- is ONE 4-d TMA box (out-of-bounds = the zero padding).
// With the tile's rows numbered on the padded pitch P = W + 2 (virtual row v = yy * P + xx,
// xx = padded column), the input of tap (dy, dx) for virtual row v is halo row
// v + (dy + 1) * P + dx: every tap is the same operand shifted by a constant number of rows,
// i.e. a descriptor start-address offset.  9 taps x 4 MMAs (K = 16) per tile read one
// 30 KB halo tile instead of 144 KB of im2col boxes; the 2 columns of padding per image row
// (v with xx = 0 or W + 1) and the tail rows v >= R * P are computed and dropped.
//   64 input channels: the halo box lands in the 128-byte-swizzled K-major layout (128-byte
//     pixel rows, one box per stage).  The swizzle is a function of the SMEM address bits, so a
//     descriptor may start at any 128-byte row of the atom (tools/sw128_shift_probe.cu: exact
//     for every row offset with base offset 0).
//   16 input channels: UMMA no-swizzle K-major planes ([rows][16 B] per 8 channels).
//   NO output channels per CTA (64 or 128); Cout = 256 (the space-to-depth stem) splits N over
//   CTA pairs: CTA b computes channels (b % 2) * 128 .. +127 of every tile it takes, so each
//   holds half the weights.
//   weights resident in SMEM (one K block per tap); ring of halo stages; TMEM double-buffered
//   accumulators; warps 0-7 epilogue (two warpgroups, alternate tiles), 8 TMA producer, 9 MMA.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>

#include "epilogue.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace dycl {
namespace {

constexpr int BM = 128;
constexpr int MAX_STAGES = 4;
constexpr int THREADS = 320;

struct HaloPlan {
  int R, P;                                  // output rows per tile, padded pitch (W + KW - 1)
  int tiles_per_sample;
  int KH, KW, padH, padW;
  int plane_rows;                            // rows per stage (per 8-channel plane when planar)
  int stages;                                // halo ring depth
  int nsplit;                                // Cout / NO: CTAs b with b % nsplit == h compute N slice h
};

template <int CH, int NO>
struct HCfg {
  static constexpr bool SW = CH == 64;       // 128-byte-swizzled pixel rows (else planar)
  static constexpr int PLANES = CH / 8;      // planar layout only
  static constexpr int KSTEPS = CH / 16;     // MMAs (K = 16) per tap
  static constexpr int B_TAP = NO * CH * 2;  // bytes of weights per tap
};

inline int halo_no(const ConvArgs& a) { return a.Cout == 64 ? 64 : 128; }

// dynamic SMEM: 1024 (align) + stages x halo stage + taps x B_TAP + barriers (256 B) + bias
inline int halo_smem(int ch, int no, const HaloPlan& hp) {
  return 1024 + hp.stages * hp.plane_rows * ch * 2 + hp.KH * hp.KW * no * ch * 2 + 256 + no * 4;
}

template <int CH, int NO, int KSZ>
__global__ void __launch_bounds__(THREADS, 1)
    k_conv_halo(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW, const ConvArgs a,
                const HaloPlan hp) {
  using Q = HCfg<CH, NO>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int PLANE = hp.plane_rows * 16;      // planar layout: bytes per 8-channel plane
  const int STAGE = hp.plane_rows * CH * 2;  // plane_rows % 8 == 0: stages stay 1024-B aligned
  constexpr int TAPS = KSZ * KSZ;
  const int S = hp.stages;
  uint8_t* sX = smem;
  uint8_t* sW = smem + S * STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sW + TAPS * Q::B_TAP);
  const uint32_t full0 = ptx::smem_u32(bars), empty0 = full0 + 8 * MAX_STAGES;
  const uint32_t tfull0 = empty0 + 8 * MAX_STAGES, tempty0 = tfull0 + 16, wfull = tempty0 + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * MAX_STAGES + 5);
  float* sBias = reinterpret_cast<float*>(sW + TAPS * Q::B_TAP + 256);     // 16-B aligned
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nh = (int)(blockIdx.x % hp.nsplit);          // this CTA's N slice
  for (int i = threadIdx.x; i < NO; i += THREADS) sBias[i] = a.bias[nh * NO + i];
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      ptx::mbar_init(full0 + 8 * i, 1);
      ptx::mbar_init(empty0 + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(tfull0 + 8 * i, 1);
      ptx::mbar_init(tempty0 + 8 * i, 128);
    }
    ptx::mbar_init(wfull, 1);
    ptx::fence_mbar_init();
  }
  constexpr uint32_t TCOLS = 2 * NO;
  if (warp == 9) ptx::tmem_alloc(ptx::smem_u32(tmem_slot), TCOLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int n_live = a.n_live ? *a.n_live : a.n_static;
  const int R = hp.R, P = hp.P, TPS = hp.tiles_per_sample;
  const int num_tiles = n_live * TPS;
  const int tile0 = (int)(blockIdx.x / hp.nsplit), tstep = (int)(gridDim.x / hp.nsplit);
  const uint32_t halo_tx = (uint32_t)((R + hp.KH - 1) * P * CH * 2);
  // K steps that can be nonzero (channels >= c_live are zero in the input and the weights)
  const int ksteps = a.c_live > 0 && a.c_live < CH ? (a.c_live + 15) / 16 : Q::KSTEPS;

  if (warp == 8) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tmX);
      ptx::tma_prefetch_desc(&tmW);
      ptx::mbar_arrive_expect_tx(wfull, (uint32_t)(TAPS * Q::B_TAP));
      if constexpr (Q::SW) {
        // weights resident, SW128: tap t -> [NO rows][128 B] at sW + t * B_TAP
        for (int t = 0; t < TAPS; ++t)
          ptx::tma_load_2d(ptx::smem_u32(sW + t * Q::B_TAP), &tmW, wfull, t * CH, nh * NO);
      } else {
        // weights resident, planar: tap t, plane p -> [NO rows][16 B] at sW + (t * PLANES + p) * NO * 16
        for (int t = 0; t < TAPS; ++t)
          for (int p = 0; p < Q::PLANES; ++p)
            ptx::tma_load_2d(ptx::smem_u32(sW + (t * Q::PLANES + p) * NO * 16), &tmW, wfull, t * CH + 8 * p,
                             nh * NO);
      }
    }
    __syncwarp();
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = tile0; tile < num_tiles; tile += tstep) {
      const int ns = tile / TPS, y0 = (tile - ns * TPS) * R;
      ptx::mbar_wait(empty0 + 8 * stage, phase ^ 1);
      if (lane == 0) {
        const uint32_t bar = full0 + 8 * stage;
        ptx::mbar_arrive_expect_tx(bar, halo_tx);
        if constexpr (Q::SW)
          ptx::tma_load_4d(ptx::smem_u32(sX + stage * STAGE), &tmX, bar, 0, -hp.padW, y0 - hp.padH, ns);
        else
          for (int p = 0; p < Q::PLANES; ++p)
            ptx::tma_load_4d(ptx::smem_u32(sX + stage * STAGE + p * PLANE), &tmX, bar, 8 * p, -hp.padW,
                             y0 - hp.padH, ns);
      }
      __syncwarp();
      if (++stage == S) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else if (warp == 9) {
    // ---------------------------------------------------------------- MMA issuer
    // Every operand address is the stage base plus a compile-time tap / K-step offset (plus
    // r * P rows): the descriptors are built once per tile and advanced by adding to their
    // start-address field (addresses < 256 KB: the 14-bit field never carries).  A per-MMA
    // descriptor build (with the tap's div / mod) cost ~40 issue slots per MMA -- longer than a
    // 128 x 64 x 16 MMA runs -- and left the tensor pipe at 27 % (ncu, round 2).
    constexpr uint32_t IDESC = ptx::make_idesc_bf16(BM, NO);
    ptx::mbar_wait(wfull, 0);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    const uint32_t pitch16 = (uint32_t)P * (Q::SW ? 8u : 1u);            // one padded image row, in 16-B units
    const uint64_t bd0 = Q::SW ? ptx::make_smem_desc_sw128(ptx::smem_u32(sW))
                               : ptx::make_smem_desc(ptx::smem_u32(sW), 0, (uint32_t)(NO * 16), 128);
    for (int tile = tile0; tile < num_tiles; tile += tstep, ++it) {
      const int acc = it & 1;
      ptx::mbar_wait(tempty0 + 8 * acc, ((it >> 1) & 1) ^ 1);
      ptx::mbar_wait(full0 + 8 * stage, phase);
      ptx::tc_fence_after();
      const uint32_t d = tmem + (uint32_t)(acc * NO);
      const uint32_t xs = ptx::smem_u32(sX + stage * STAGE);
      const uint64_t ad0 = Q::SW ? ptx::make_smem_desc_sw128(xs) : ptx::make_smem_desc(xs, 0, (uint32_t)PLANE, 128);
      if (ptx::elect_one()) {
        const uint32_t alo = (uint32_t)ad0, ahi = (uint32_t)(ad0 >> 32);
        const uint32_t blo = (uint32_t)bd0, bhi = (uint32_t)(bd0 >> 32);
#pragma unroll 1
        for (int r = 0; r < KSZ; ++r) {
          const uint32_t alr = alo + (uint32_t)r * pitch16;
          const uint32_t blr = blo + (uint32_t)(r * KSZ) * (Q::SW ? Q::B_TAP >> 4 : Q::PLANES * NO);
#pragma unroll
          for (int s = 0; s < KSZ; ++s) {
#pragma unroll
            for (int j = 0; j < Q::KSTEPS; ++j) {
              // SW: row shift inside the swizzle atom = start address only (base offset 0); K step j = +32 B.
              // planar: K step j = channels 16j .. 16j+15 = planes 2j, 2j+1 (LBO = plane stride, SBO = 8 rows)
              const uint32_t a_off = Q::SW ? s * 8 + 2 * j : s + 2 * j * (PLANE >> 4);
              const uint32_t b_off = Q::SW ? s * (Q::B_TAP >> 4) + 2 * j : (s * Q::PLANES + 2 * j) * NO;
              if (j < ksteps) ptx::mma_bf16_ss_lohi(d, alr + a_off, ahi, blr + b_off, bhi, IDESC, (r | s | j) != 0);
            }
          }
        }
      }
      __syncwarp();
      ptx::mma_commit_elect(empty0 + 8 * stage);
      ptx::mma_commit_elect(tfull0 + 8 * acc);
      __syncwarp();
      if (++stage == S) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    const int wg = warp >> 2, quad = warp & 3;
    const int v = quad * 32 + lane;                       // virtual row of the tile
    const int yy = v / P, xx = v - (v / P) * P;
    const bool real = xx < a.Wo && yy < R;
    int it = 0;
    for (int tile = tile0; tile < num_tiles; tile += tstep, ++it) {
      if ((it & 1) != wg) continue;
      const int acc = it & 1;
      const int ns = tile / TPS, y0 = (tile - ns * TPS) * R;
      ptx::mbar_wait(tfull0 + 8 * acc, (it >> 1) & 1);
      ptx::tc_fence_after();
      const uint32_t tb = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * NO);
      uint16_t* out = a.y + (((size_t)ns * a.Ho + (y0 + yy)) * a.Wo + xx) * a.Cout + nh * NO;
#pragma unroll 1
      for (int c0 = 0; c0 < NO; c0 += 32) {
        uint32_t t16[2][16];
        ptx::tmem_ld_32x32b_x16(tb + (uint32_t)c0, t16[0]);
        ptx::tmem_ld_32x32b_x16(tb + (uint32_t)c0 + 16, t16[1]);
        float bv[32];
#pragma unroll
        for (int q = 0; q < 32; q += 4) {
          const float4 b4 = *reinterpret_cast<const float4*>(sBias + c0 + q);
          bv[q] = b4.x; bv[q + 1] = b4.y; bv[q + 2] = b4.z; bv[q + 3] = b4.w;
        }
        ptx::tmem_ld_wait();
        if (real) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float f[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              f[q] = __uint_as_float(t16[h][q]) + bv[16 * h + q];
              if (a.relu) f[q] = fmaxf(f[q], 0.f);
            }
            uint4* o = reinterpret_cast<uint4*>(out + c0 + 16 * h);
            o[0] = make_uint4(pack_bf16x2_rn(f[0], f[1]), pack_bf16x2_rn(f[2], f[3]), pack_bf16x2_rn(f[4], f[5]),
                              pack_bf16x2_rn(f[6], f[7]));
            o[1] = make_uint4(pack_bf16x2_rn(f[8], f[9]), pack_bf16x2_rn(f[10], f[11]), pack_bf16x2_rn(f[12], f[13]),
                              pack_bf16x2_rn(f[14], f[15]));
          }
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(tempty0 + 8 * acc);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, TCOLS);
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn_halo() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

bool halo_plan(const ConvArgs& a, HaloPlan* hp) {
  hp->KH = hp->KW = a.ksz;
  hp->padH = hp->padW = a.pad;
  // output x reads input columns x - pad .. x - pad + ksz - 1 (out of range = zero padding, on
  // either side: the TMA box's out-of-bounds fill), so a tile row spans P = Wo + ksz - 1 columns
  const int P = a.Wo + a.ksz - 1;
  if (P > 256 || a.Ho < 1 || a.Wo < 1) return false;
  int R = 0;
  for (int r = 1; r <= a.Ho; ++r)
    if (a.Ho % r == 0 && r * P <= BM) R = r;
  // >= 75 % of the 128 MMA rows real (small maps -- e.g. 8 x 8, 80 of 128 -- keep the GEMM's
  // whole-sample row-tap form)
  if (R == 0 || R * a.Wo < 96 || R + a.ksz - 1 > 256) return false;
  // rows per stage: the halo, and the furthest row an MMA row reads (tap (KH-1, KW-1) of row 127)
  const int rows = std::max((R + a.ksz - 1) * P, BM + (a.ksz - 1) * P + (a.ksz - 1));
  hp->R = R;
  hp->P = P;
  hp->tiles_per_sample = a.Ho / R;
  hp->plane_rows = (rows + 7) / 8 * 8;
  const int no = halo_no(a);
  hp->nsplit = a.Cout / no;
  for (hp->stages = MAX_STAGES; hp->stages >= 2; --hp->stages)
    if (halo_smem(a.C, no, *hp) <= 227 * 1024) return true;
  return false;
}

}  // namespace

bool conv_halo_eligible(const ConvArgs& a) {
  HaloPlan hp;
  const bool shape = (a.C == 64 && a.ksz == 3 && (a.Cout == 64 || a.Cout == 128 || a.Cout == 256)) ||
                     (a.C == 16 && a.ksz == 4 && a.Cout == 64);
  return a.in_nhwc && a.nhwc && a.stride == 1 && shape && a.Kp == a.ksz * a.ksz * a.C && a.res_mode == 0 && !a.y32 && !a.x2 && !a.rows_in && !a.rows_out &&
         !a.gap_part && !a.rows_gather && a.y && !(a.dbg & 8388608) && halo_plan(a, &hp);
}

template <int CH, int NO, int KSZ>
cudaError_t launch_ch(const ConvArgs& a, const HaloPlan& hp, int max_rows, int num_sms, cudaStream_t stream) {
  using Q = HCfg<CH, NO>;
  EncodeTiledFn enc = encode_fn_halo();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap tmX, tmW;
  {
    const int rows = max_rows > 0 ? max_rows : 1;
    cuuint64_t dims[4] = {(cuuint64_t)CH, (cuuint64_t)a.W, (cuuint64_t)a.H, (cuuint64_t)rows};
    cuuint64_t strides[3] = {(cuuint64_t)CH * 2, (cuuint64_t)a.W * CH * 2, (cuuint64_t)a.H * a.W * CH * 2};
    cuuint32_t box[4] = {Q::SW ? (cuuint32_t)CH : 8u, (cuuint32_t)hp.P, (cuuint32_t)(hp.R + hp.KH - 1), 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (enc(&tmX, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, (void*)a.x, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, Q::SW ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    cuuint64_t dims[2] = {(cuuint64_t)a.Kp, (cuuint64_t)a.Cout};
    cuuint64_t strides[1] = {(cuuint64_t)a.Kp * 2};
    cuuint32_t box[2] = {Q::SW ? (cuuint32_t)CH : 8u, (cuuint32_t)NO};
    cuuint32_t es[2] = {1, 1};
    if (enc(&tmW, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void*)a.w, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, Q::SW ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  const int smem = halo_smem(CH, NO, hp);
  if (cudaError_t e = ensure_smem(k_conv_halo<CH, NO, KSZ>, smem)) return e;
  const long long tiles = (long long)(max_rows > 0 ? max_rows : 1) * hp.tiles_per_sample * hp.nsplit;
  int grid = (int)(tiles < num_sms ? tiles : num_sms);
  grid -= grid % hp.nsplit;                 // whole CTA groups: every N slice sees every tile
  if (grid < hp.nsplit) grid = hp.nsplit;
  return launch_k(k_conv_halo<CH, NO, KSZ>, dim3(grid), dim3(THREADS), (size_t)smem, stream, tmX, tmW, a, hp);
}

cudaError_t launch_conv_halo(const ConvArgs& a, int max_rows, int num_sms, cudaStream_t stream) {
  HaloPlan hp;
  if (!conv_halo_eligible(a) || !halo_plan(a, &hp)) return cudaErrorNotSupported;
  if (a.C == 16) return launch_ch<16, 64, 4>(a, hp, max_rows, num_sms, stream);
  if (a.Cout == 64) return launch_ch<64, 64, 3>(a, hp, max_rows, num_sms, stream);
  return launch_ch<64, 128, 3>(a, hp, max_rows, num_sms, stream);
}

// Lazy-loading anchor: a kernel of this translation unit's module (preload_kernels, hostmod.cu).
__global__ void k_tu_anchor_conv_halo() {}
const void* tu_anchor_conv_halo() { return reinterpret_cast<const void*>(&k_tu_anchor_conv_halo); }

}  // namespace dycl
