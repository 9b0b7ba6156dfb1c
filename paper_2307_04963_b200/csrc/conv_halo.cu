// KxK / stride-1 NHWC convolution with a TMA halo tile and shifted UMMA descriptors
// (the ResNet-50 stage-1 bottleneck conv2, 3x3 56x56x64 -> 64, and the stem in
// its 2x2 space-to-depth form, 4x4 over 112x112x16 -> 64).
//
// The im2col GEMM (conv_gemm.cu) loads one TMA im2col box per tap: 9 x 16 KB of A per 128-row
// tile, and on the 64-channel 3x3 layers that operand feed (not the tensor core) bounds it
// (ncu: tensor pipe 26 %, producer / full-barrier waits on top; profiles/r02_ncu_conv_gemm_cfg5.txt).
// Here a tile is R whole output rows of one sample.  Its input with the 1-pixel halo -- rows
// y0-1 .. y0+R, columns -1 .. W -- is ONE 4-d TMA box per 8-channel plane (out-of-bounds = the
// zero padding), landing in SMEM in the UMMA no-swizzle K-major layout: plane p = [rows][16 B].
// With the tile's rows numbered on the padded pitch P = W + 2 (virtual row v = yy * P + xx,
// xx = padded column), the input of tap (dy, dx) for virtual row v is halo row
// v + (dy + 1) * P + dx: every tap is the same operand shifted by a constant number of 16-byte
// rows, i.e. a descriptor start-address offset.  9 taps x 4 MMAs (K = 16) per tile read one
// 30 KB halo tile instead of 144 KB of im2col boxes; the 2 columns of padding per image row
// (v with xx = 0 or W + 1) and the tail rows v >= R * P are computed and dropped.
//   weights: [64][9 * 64] bf16 resident in SMEM (SW128, one K block per tap)
//   warps 0-7 epilogue (two warpgroups, alternate tiles), 8 TMA producer, 9 MMA.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>

#include "epilogue.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace dycl {
namespace {

constexpr int BM = 128;
constexpr int NO = 64;                      // output channels (N)
constexpr int STAGES = 4;
constexpr int THREADS = 320;

struct HaloPlan {
  int R, P;                                  // output rows per tile, padded pitch (W + KW - 1)
  int tiles_per_sample;
  int KH, KW, padH, padW;
  int plane_rows;                            // rows per 8-channel plane per stage
};

template <int CH>
struct HCfg {
  static constexpr int PLANES = CH / 8;
  static constexpr int KSTEPS = CH / 16;     // MMAs (K = 16) per tap
  static constexpr int B_TAP = NO * CH * 2;  // bytes of weights per tap (planar: [CH/8][NO][16 B])
};

// dynamic SMEM: 1024 (align) + STAGES x halo stage + taps x B_TAP + barriers
inline int halo_smem(int ch, const HaloPlan& hp) {
  return 1024 + STAGES * (ch / 8) * hp.plane_rows * 16 + hp.KH * hp.KW * NO * ch * 2 + 256;
}

template <int CH>
__global__ void __launch_bounds__(THREADS, 1)
    k_conv_halo(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW, const ConvArgs a,
                const HaloPlan hp) {
  using Q = HCfg<CH>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int PLANE = hp.plane_rows * 16;
  const int STAGE = Q::PLANES * PLANE;
  const int TAPS = hp.KH * hp.KW;
  uint8_t* sX = smem;
  uint8_t* sW = smem + STAGES * STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sW + TAPS * Q::B_TAP);
  const uint32_t full0 = ptx::smem_u32(bars), empty0 = full0 + 8 * STAGES;
  const uint32_t tfull0 = empty0 + 8 * STAGES, tempty0 = tfull0 + 16, wfull = tempty0 + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 5);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
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
  if (warp == 9) ptx::tmem_alloc(ptx::smem_u32(tmem_slot), 128);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int n_live = a.n_live ? *a.n_live : a.n_static;
  const int R = hp.R, P = hp.P, TPS = hp.tiles_per_sample;
  const int num_tiles = n_live * TPS;
  const uint32_t halo_tx = (uint32_t)(Q::PLANES * (R + hp.KH - 1) * P * 16);

  if (warp == 8) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tmX);
      ptx::tma_prefetch_desc(&tmW);
      // weights resident, planar: tap t, plane p -> [NO rows][16 B] at sW + (t * PLANES + p) * NO * 16
      ptx::mbar_arrive_expect_tx(wfull, (uint32_t)(TAPS * Q::B_TAP));
      for (int t = 0; t < TAPS; ++t)
        for (int p = 0; p < Q::PLANES; ++p)
          ptx::tma_load_2d(ptx::smem_u32(sW + (t * Q::PLANES + p) * NO * 16), &tmW, wfull, t * CH + 8 * p, 0);
    }
    __syncwarp();
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int ns = tile / TPS, y0 = (tile - ns * TPS) * R;
      ptx::mbar_wait(empty0 + 8 * stage, phase ^ 1);
      if (lane == 0) {
        const uint32_t bar = full0 + 8 * stage;
        ptx::mbar_arrive_expect_tx(bar, halo_tx);
        for (int p = 0; p < Q::PLANES; ++p)
          ptx::tma_load_4d(ptx::smem_u32(sX + stage * STAGE + p * PLANE), &tmX, bar, 8 * p, -hp.padW, y0 - hp.padH, ns);
      }
      __syncwarp();
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else if (warp == 9) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t IDESC = ptx::make_idesc_bf16(BM, NO);
    ptx::mbar_wait(wfull, 0);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      ptx::mbar_wait(tempty0 + 8 * acc, ((it >> 1) & 1) ^ 1);
      ptx::mbar_wait(full0 + 8 * stage, phase);
      ptx::tc_fence_after();
      const uint32_t d = tmem + (uint32_t)(acc * NO);
      const uint32_t xs = ptx::smem_u32(sX + stage * STAGE);
      const uint32_t ws = ptx::smem_u32(sW);
#pragma unroll 1
      for (int t = 0; t < TAPS; ++t) {
        const int r = t / hp.KW, s = t - r * hp.KW;
        const uint32_t row0 = (uint32_t)(r * P + s);                      // tap (r - padH, s - padW)
#pragma unroll
        for (int j = 0; j < Q::KSTEPS; ++j) {
          // K step j = channels 16j .. 16j+15 = planes 2j, 2j+1 (LBO = plane stride, SBO = 8 rows)
          const uint64_t ad = ptx::make_smem_desc(xs + (uint32_t)(2 * j * PLANE) + row0 * 16, 0, (uint32_t)PLANE, 128);
          const uint64_t bd =
              ptx::make_smem_desc(ws + (uint32_t)((t * Q::PLANES + 2 * j) * NO * 16), 0, (uint32_t)(NO * 16), 128);
          ptx::mma_bf16_ss_elect(d, ad, bd, IDESC, (uint32_t)((t | j) != 0));
        }
      }
      ptx::mma_commit_elect(empty0 + 8 * stage);
      ptx::mma_commit_elect(tfull0 + 8 * acc);
      __syncwarp();
      if (++stage == STAGES) {
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
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      if ((it & 1) != wg) continue;
      const int acc = it & 1;
      const int ns = tile / TPS, y0 = (tile - ns * TPS) * R;
      ptx::mbar_wait(tfull0 + 8 * acc, (it >> 1) & 1);
      ptx::tc_fence_after();
      const uint32_t tb = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * NO);
      uint16_t* out = a.y + (((size_t)ns * a.Ho + (y0 + yy)) * a.Wo + xx) * NO;
#pragma unroll 1
      for (int c0 = 0; c0 < NO; c0 += 16) {
        uint32_t t16[16];
        ptx::tmem_ld_32x32b_x16(tb + (uint32_t)c0, t16);
        ptx::tmem_ld_wait();
        if (real) {
          float f[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            f[q] = __uint_as_float(t16[q]) + __ldg(a.bias + c0 + q);
            if (a.relu) f[q] = fmaxf(f[q], 0.f);
          }
          uint4* o = reinterpret_cast<uint4*>(out + c0);
          o[0] = make_uint4(pack_bf16x2_rn(f[0], f[1]), pack_bf16x2_rn(f[2], f[3]), pack_bf16x2_rn(f[4], f[5]),
                            pack_bf16x2_rn(f[6], f[7]));
          o[1] = make_uint4(pack_bf16x2_rn(f[8], f[9]), pack_bf16x2_rn(f[10], f[11]), pack_bf16x2_rn(f[12], f[13]),
                            pack_bf16x2_rn(f[14], f[15]));
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
    ptx::tmem_dealloc(tmem, 128);
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
  if (R == 0 || R * a.Wo < 96) return false;
  // rows per plane: the halo, and the furthest row an MMA row reads (tap (KH-1, KW-1) of row 127)
  const int rows = std::max((R + a.ksz - 1) * P, BM + (a.ksz - 1) * P + (a.ksz - 1));
  hp->R = R;
  hp->P = P;
  hp->tiles_per_sample = a.Ho / R;
  hp->plane_rows = (rows + 7) / 8 * 8;
  const int smem = halo_smem(a.C, *hp);
  return smem <= 227 * 1024;
}

}  // namespace

bool conv_halo_eligible(const ConvArgs& a) {
  HaloPlan hp;
  return a.in_nhwc && a.nhwc && a.stride == 1 && (a.C == 64 || a.C == 16) && a.Cout == NO &&
         a.Kp == a.ksz * a.ksz * a.C && (a.ksz == 3 || a.ksz == 4) && a.res_mode == 0 && !a.y32 && !a.x2 &&
         !a.rows_in && !a.rows_out && !a.gap_part && !a.rows_gather && a.y && !(a.dbg & 8388608) &&
         halo_plan(a, &hp);
}

template <int CH>
cudaError_t launch_ch(const ConvArgs& a, const HaloPlan& hp, int max_rows, int num_sms, cudaStream_t stream) {
  EncodeTiledFn enc = encode_fn_halo();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap tmX, tmW;
  {
    const int rows = max_rows > 0 ? max_rows : 1;
    cuuint64_t dims[4] = {(cuuint64_t)CH, (cuuint64_t)a.W, (cuuint64_t)a.H, (cuuint64_t)rows};
    cuuint64_t strides[3] = {(cuuint64_t)CH * 2, (cuuint64_t)a.W * CH * 2, (cuuint64_t)a.H * a.W * CH * 2};
    cuuint32_t box[4] = {8, (cuuint32_t)hp.P, (cuuint32_t)(hp.R + hp.KH - 1), 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (enc(&tmX, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, (void*)a.x, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    cuuint64_t dims[2] = {(cuuint64_t)a.Kp, (cuuint64_t)NO};
    cuuint64_t strides[1] = {(cuuint64_t)a.Kp * 2};
    cuuint32_t box[2] = {8, (cuuint32_t)NO};
    cuuint32_t es[2] = {1, 1};
    if (enc(&tmW, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void*)a.w, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  const int smem = halo_smem(CH, hp);
  if (cudaError_t e = ensure_smem(k_conv_halo<CH>, smem)) return e;
  const long long tiles = (long long)(max_rows > 0 ? max_rows : 1) * hp.tiles_per_sample;
  int grid = (int)(tiles < num_sms ? tiles : num_sms);
  if (grid < 1) grid = 1;
  return launch_k(k_conv_halo<CH>, dim3(grid), dim3(THREADS), (size_t)smem, stream, tmX, tmW, a, hp);
}

cudaError_t launch_conv_halo(const ConvArgs& a, int max_rows, int num_sms, cudaStream_t stream) {
  HaloPlan hp;
  if (!conv_halo_eligible(a) || !halo_plan(a, &hp)) return cudaErrorNotSupported;
  return a.C == 64 ? launch_ch<64>(a, hp, max_rows, num_sms, stream) : launch_ch<16>(a, hp, max_rows, num_sms, stream);
}

}  // namespace dycl
