// 3x3 / stride-1 / pad-1 NHWC convolution with a TMA halo tile and shifted UMMA descriptors
// (the ResNet-50 stage-1 bottleneck conv2, 56x56x64 -> 64).
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

#include "epilogue.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace dycl {
namespace {

constexpr int BM = 128;
constexpr int CH = 64;                      // input channels (one K block per tap)
constexpr int NO = 64;                      // output channels (N)
constexpr int PLANES = CH / 8;
constexpr int PLANE_ROWS = 256;             // rows per plane per stage (halo + lead / tail slack)
constexpr int LEAD = 8;                     // halo starts at plane row 8 (tap offsets >= -1)
constexpr int PLANE = PLANE_ROWS * 16;      // bytes
constexpr int STAGE = PLANES * PLANE;       // 32 KB
constexpr int STAGES = 4;
constexpr int B_TAP = NO * CH * 2;          // 8 KB per tap
constexpr int B_BYTES = 9 * B_TAP;          // 72 KB
constexpr int THREADS = 320;
constexpr int SMEM = 1024 + STAGES * STAGE + B_BYTES + 256;

struct HaloPlan {
  int R, P;                                  // output rows per tile, padded pitch
  int tiles_per_sample;
};

__global__ void __launch_bounds__(THREADS, 1)
    k_conv_halo(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW, const ConvArgs a,
                const HaloPlan hp) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sX = smem;
  uint8_t* sW = smem + STAGES * STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sW + B_BYTES);
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
  const uint32_t halo_tx = (uint32_t)(PLANES * (R + 2) * P * 16);

  if (warp == 8) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tmX);
      ptx::tma_prefetch_desc(&tmW);
      ptx::mbar_arrive_expect_tx(wfull, (uint32_t)B_BYTES);
      for (int t = 0; t < 9; ++t) ptx::tma_load_2d(ptx::smem_u32(sW + t * B_TAP), &tmW, wfull, t * CH, 0);
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
        for (int p = 0; p < PLANES; ++p)
          ptx::tma_load_4d(ptx::smem_u32(sX + stage * STAGE + p * PLANE + LEAD * 16), &tmX, bar, 8 * p, -1, y0 - 1, ns);
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
#pragma unroll 1
      for (int t = 0; t < 9; ++t) {
        const int r = t / 3, s = t - 3 * (t / 3);
        const uint32_t row0 = (uint32_t)(LEAD + r * P + s - 1);          // tap (r - 1, s - 1)
        const uint64_t bd = ptx::make_smem_desc_sw128(ptx::smem_u32(sW + t * B_TAP));
#pragma unroll
        for (int j = 0; j < CH / 16; ++j) {
          // K step j = channels 16j .. 16j+15 = planes 2j, 2j+1 (LBO = plane stride, SBO = 8 rows)
          const uint64_t ad = ptx::make_smem_desc(xs + (uint32_t)(2 * j * PLANE) + row0 * 16, 0, PLANE, 128);
          ptx::mma_bf16_ss_elect(d, ad, bd + (uint64_t)(2 * j), IDESC, (uint32_t)((t | j) != 0));
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
    const bool real_col = xx >= 1 && xx <= P - 2 && yy < R;
    int it = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      if ((it & 1) != wg) continue;
      const int acc = it & 1;
      const int ns = tile / TPS, y0 = (tile - ns * TPS) * R;
      ptx::mbar_wait(tfull0 + 8 * acc, (it >> 1) & 1);
      ptx::tc_fence_after();
      const uint32_t tb = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * NO);
      uint16_t* out = a.y + (((size_t)ns * a.Ho + (y0 + yy)) * a.Wo + (xx - 1)) * NO;
#pragma unroll 1
      for (int c0 = 0; c0 < NO; c0 += 16) {
        uint32_t t16[16];
        ptx::tmem_ld_32x32b_x16(tb + (uint32_t)c0, t16);
        ptx::tmem_ld_wait();
        if (real_col) {
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
  const int P = a.W + 2;
  if (P > BM || a.H < 1) return false;
  int R = 0;
  for (int r = 1; r <= a.H; ++r)
    if (a.H % r == 0 && r * P <= BM) R = r;
  // the halo rows and the furthest row any MMA row reads (tap (1, 1) of virtual row 127) fit a plane
  if (R == 0 || LEAD + (R + 2) * P > PLANE_ROWS || LEAD + 2 * P + BM >= PLANE_ROWS) return false;
  // >= 75 % of the 128 MMA rows real (small maps -- e.g. 8 x 8, 80 of 128 -- keep the GEMM's
  // whole-sample row-tap form)
  if (R * a.W < 96) return false;
  hp->R = R;
  hp->P = P;
  hp->tiles_per_sample = a.H / R;
  return true;
}

}  // namespace

bool conv_halo_eligible(const ConvArgs& a) {
  HaloPlan hp;
  return a.in_nhwc && a.nhwc && a.ksz == 3 && a.stride == 1 && a.pad == 1 && a.C == CH && a.Cout == NO &&
         a.Kp == 9 * CH && a.Ho == a.H && a.Wo == a.W && a.res_mode == 0 && !a.y32 && !a.x2 && !a.rows_in &&
         !a.rows_out && !a.gap_part && a.y && !(a.dbg & 8388608) && halo_plan(a, &hp);
}

cudaError_t launch_conv_halo(const ConvArgs& a, int max_rows, int num_sms, cudaStream_t stream) {
  HaloPlan hp;
  if (!conv_halo_eligible(a) || !halo_plan(a, &hp)) return cudaErrorNotSupported;
  EncodeTiledFn enc = encode_fn_halo();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap tmX, tmW;
  {
    const int rows = max_rows > 0 ? max_rows : 1;
    cuuint64_t dims[4] = {(cuuint64_t)CH, (cuuint64_t)a.W, (cuuint64_t)a.H, (cuuint64_t)rows};
    cuuint64_t strides[3] = {(cuuint64_t)CH * 2, (cuuint64_t)a.W * CH * 2, (cuuint64_t)a.H * a.W * CH * 2};
    cuuint32_t box[4] = {8, (cuuint32_t)hp.P, (cuuint32_t)(hp.R + 2), 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (enc(&tmX, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, (void*)a.x, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    cuuint64_t dims[2] = {(cuuint64_t)a.Kp, (cuuint64_t)NO};
    cuuint64_t strides[1] = {(cuuint64_t)a.Kp * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)NO};
    cuuint32_t es[2] = {1, 1};
    if (enc(&tmW, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void*)a.w, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  if (cudaError_t e = ensure_smem(k_conv_halo, SMEM)) return e;
  const long long tiles = (long long)(max_rows > 0 ? max_rows : 1) * hp.tiles_per_sample;
  int grid = (int)(tiles < num_sms ? tiles : num_sms);
  if (grid < 1) grid = 1;
  return launch_k(k_conv_halo, dim3(grid), dim3(THREADS), SMEM, stream, tmX, tmW, a, hp);
}

}  // namespace dycl
