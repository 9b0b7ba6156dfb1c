// TMA-fed implicit-GEMM convolution / dense layer on tcgen05 (sm_100a) -- the
// fast path of SURVEY §8(a) a1 for every layer whose output rows tile as
// rectangular boxes (all CIFAR ResNet / MLP layers).
//
//   D[m, o] = sum_k A[m, k] B[o, k],  m = output pixel, k = (tap r,s ; channel c)
//
// Implicit GEMM without an im2col buffer: for a tile of output pixels that forms a
// box (bn samples x bh output rows x Wo columns, <= 128 rows) the A operand of one
// filter tap (r, s) is itself a 4-D box of the NHWC input
//     x[n0 .. n0+bn)[ho0*st-pad+r :: st][-pad+s :: st][c0 .. c0+CW)
// which ONE TMA instruction fetches (negative / past-the-end coordinates are
// zero-filled by the TMA unit: that is the convolution's zero padding; the
// traversal stride implements stride 2).  The box lands as 128 K-major rows of
// CW channels in the UMMA canonical layout whose swizzle equals the row width
// (32/64/128 B), so each TMA box feeds CW/16 tcgen05.mma K-steps directly.
//
// Warp roles (persistent CTA per SM, 6 warps):
//   warps 0-3  epilogue: tcgen05.ld -> +bias, +shortcut (identity / option A,
//              bf16 or fp32 residual stream), ReLU, RNE->bf16 (+ fp32 copy)
//   warp  4    TMA producer (one elected lane): weights once (resident in smem),
//              then one A box per (tile, tap, channel chunk) into a deep ring
//   warp  5    TMEM allocator + MMA issuer (one lane), double-buffered accumulator
#include <cuda.h>
#include <cuda_bf16.h>

#include "kernels.h"
#include "ptx.cuh"

namespace dycl {
namespace {

constexpr int BM = 128;
constexpr int THREADS = 192;
constexpr int SMEM_BUDGET = 200 * 1024;

// K is cut into "units": one (tap, channel chunk) = one TMA box of CW channels.
// A ring stage holds U units (amortising the per-stage mbarrier handshakes over
// several taps); a tile takes nks = ceil(nunits / U) stages.
struct TmaGeom {
  int CW;            // channels per unit (box inner dimension)
  int cchunks;       // C / CW
  int nunits;        // ksz*ksz*cchunks (even for C == 8: phantom zero unit appended)
  int U;             // units per ring stage
  int nks;           // ring stages per tile
  int layout;        // UMMA layout code (0 none, 2/4/6 = 128/64/32-byte swizzle)
  int row_bytes;     // bytes of one row of a unit (CW * 2)
  int unit_bytes;    // A smem per unit: 128 rows
  int b_unit_bytes;  // B smem per unit: BN rows
  int bn, bh, rows;  // tile box: samples x output rows; rows = bn*bh*Wo
};

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

struct TmaParams {
  ConvArgs a;
  TmaGeom g;
  int stages;
  int tiles_per_img_group;   // tiles covering one group of bn samples
};

template <int BN>
__global__ void __launch_bounds__(THREADS, 1)
    k_conv_tma(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const TmaParams P) {
  const ConvArgs& a = P.a;
  const TmaGeom& G = P.g;
  const int S = P.stages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int n_tiles = a.Cout / BN;
  uint8_t* sB = smem;                                         // resident weights [n_tiles][nunits][BN rows]
  const int b_total = (G.nunits * G.b_unit_bytes * n_tiles + 1023) & ~1023;
  const int a_stage_bytes = G.U * G.unit_bytes;
  uint8_t* sA = smem + b_total;                               // ring: S stages x U units
  uint64_t* bars = reinterpret_cast<uint64_t*>(sA + S * a_stage_bytes);
  const uint32_t full0 = ptx::smem_u32(bars);
  const uint32_t empty0 = full0 + 8 * S;
  const uint32_t tfull0 = empty0 + 8 * S;
  const uint32_t tempty0 = tfull0 + 16;
  const uint32_t bfull = tempty0 + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 5);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_live = a.n_live ? *a.n_live : a.n_static;
  const int groups = (n_live + G.bn - 1) / G.bn;             // sample groups of bn
  const int m_tiles = groups * P.tiles_per_img_group;
  const int num_tiles = m_tiles * n_tiles;
  constexpr int TMEM_COLS = (2 * BN) <= 32 ? 32 : (2 * BN) <= 64 ? 64 : (2 * BN) <= 128 ? 128 : (2 * BN) <= 256 ? 256 : 512;

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      ptx::mbar_init(full0 + 8 * i, 1);
      ptx::mbar_init(empty0 + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(tfull0 + 8 * i, 1);
      ptx::mbar_init(tempty0 + 8 * i, 128);
    }
    ptx::mbar_init(bfull, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 5) ptx::tmem_alloc(ptx::smem_u32(tmem_slot), TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int taps = a.ksz * a.ksz;
  if (warp == 4) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tmA);
      ptx::tma_prefetch_desc(&tmB);
      // Weights of every unit of every N tile: resident for the whole persistent loop.
      ptx::mbar_arrive_expect_tx(bfull, (uint32_t)(G.nunits * G.b_unit_bytes * n_tiles));
      for (int nt = 0; nt < n_tiles; ++nt)
        for (int u = 0; u < G.nunits; ++u) {
          const uint32_t dst = ptx::smem_u32(sB + (nt * G.nunits + u) * G.b_unit_bytes);
          const int tap = u / G.cchunks, cc = u - tap * G.cchunks;
          ptx::tma_load_2d(dst, &tmB, bfull, tap * a.C + cc * G.CW, nt * BN);   // phantom tap: zero weights
        }
      const uint32_t unit_tx = (uint32_t)(G.rows * G.row_bytes);
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int m_tile = tile / n_tiles;
        const int grp = m_tile / P.tiles_per_img_group;
        const int ho0 = (m_tile - grp * P.tiles_per_img_group) * G.bh;
        const int n0 = grp * G.bn;
        const int h0 = ho0 * a.stride - a.pad;
        const int w0 = -a.pad;
        int r = 0, sc = 0, cc = 0, tap = 0;     // running (tap row, tap col, channel chunk)
        for (int ks = 0; ks < G.nks; ++ks) {
          const int nu = min(G.U, G.nunits - ks * G.U);
          ptx::mbar_wait(empty0 + 8 * stage, phase ^ 1);
          const uint32_t bar = full0 + 8 * stage;
          if (a.dbg & 4) {
            ptx::mbar_arrive(bar);
            if (++stage == S) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          ptx::mbar_arrive_expect_tx(bar, unit_tx * (uint32_t)nu);
          uint32_t dst = ptx::smem_u32(sA + stage * a_stage_bytes);
          for (int u = 0; u < nu; ++u, dst += G.unit_bytes) {
            // phantom tap (C == 8 padding to an even unit count): fully out of range -> zeros
            const int hh = tap < taps ? h0 + r : -(1 << 20);
            ptx::tma_load_4d(dst, &tmA, bar, cc * G.CW, w0 + sc, hh, n0);
            if (++cc == G.cchunks) {
              cc = 0;
              ++tap;
              if (++sc == a.ksz) {
                sc = 0;
                ++r;
              }
            }
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 5) {
    // ---------------------------------------------------------------- MMA issuer
    const uint32_t IDESC = ptx::make_idesc_bf16(BM, BN);
    const bool pair = G.CW == 8;                               // 16-byte rows: a K-step spans two units
    const int ksteps_unit = pair ? 1 : G.CW / 16;
    const uint32_t a_sbo = pair ? 128u : (uint32_t)(8 * G.row_bytes);
    const uint32_t a_lbo = pair ? (uint32_t)G.unit_bytes : 16u;
    const uint32_t b_lbo = pair ? (uint32_t)G.b_unit_bytes : 16u;
    const uint64_t adesc0 = ptx::make_smem_desc(ptx::smem_u32(sA), G.layout, a_lbo, a_sbo);
    const uint64_t bdesc0 = ptx::make_smem_desc(ptx::smem_u32(sB), G.layout, b_lbo, a_sbo);
    ptx::mbar_wait(bfull, 0);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int n_tile = tile % n_tiles;
      ptx::mbar_wait(tempty0 + 8 * acc, acc_phase ^ 1);
      ptx::tc_fence_after();
      const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
      uint32_t b_off = (uint32_t)(n_tile * G.nunits * G.b_unit_bytes);
      for (int ks = 0; ks < G.nks; ++ks) {
        const int nu = min(G.U, G.nunits - ks * G.U);
        ptx::mbar_wait(full0 + 8 * stage, phase);
        ptx::tc_fence_after();
        if (lane == 0) {
          uint32_t a_off = (uint32_t)(stage * a_stage_bytes);
          const int step_units = pair ? 2 : 1;
          for (int u = 0; u < nu && !(a.dbg & 2); u += step_units) {
            for (int j = 0; j < ksteps_unit; ++j) {
              ptx::mma_bf16_ss(d_tmem, adesc0 + ((a_off + 32 * j) >> 4), bdesc0 + ((b_off + 32 * j) >> 4), IDESC,
                               (ks | u | j) != 0);
            }
            a_off += step_units * G.unit_bytes;
            b_off += step_units * G.b_unit_bytes;
          }
          ptx::mma_commit(empty0 + 8 * stage);
        }
        if (lane != 0) b_off += (uint32_t)(nu * G.b_unit_bytes);
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
    // ---------------------------------------------------------------- epilogue
    const int row = warp * 32 + lane;
    const int img_rows = G.bh * a.Wo;                          // rows of one sample inside the tile box
    const int HoWo = a.Ho * a.Wo;
    int it = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int m_tile = tile / n_tiles;
      const int n_tile = tile - m_tile * n_tiles;
      const int grp = m_tile / P.tiles_per_img_group;
      const int ho0 = (m_tile - grp * P.tiles_per_img_group) * G.bh;
      const int nn = row / img_rows;
      const int rr = row - nn * img_rows;
      const int n = grp * G.bn + nn;
      const int ho = ho0 + rr / a.Wo;
      const int wo = rr - (rr / a.Wo) * a.Wo;
      const bool ok = row < G.rows && n < n_live && ho < a.Ho;
      const size_t m = (size_t)n * HoWo + (size_t)ho * a.Wo + wo;   // output pixel (row of y)
      ptx::mbar_wait(tfull0 + 8 * acc, acc_phase);
      ptx::tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(warp * 32) << 16) + (uint32_t)(acc * BN);
      size_t rbase = 0;
      if (a.res_mode == 1) rbase = m * a.Cout;
      else if (a.res_mode == 2) rbase = (((size_t)n * a.rH + 2 * ho) * a.rW + 2 * wo) * a.rC;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t v[16];
        ptx::tmem_ld_32x32b_x16(taddr + (uint32_t)c0, v);
        ptx::tmem_ld_wait();
        if (ok && !(a.dbg & 1)) {
          const int o0 = n_tile * BN + c0;
          float f[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) f[j] = __uint_as_float(v[j]) + __ldg(a.bias + o0 + j);
          if (a.res_mode == 1) {
            if (a.res32) {
              const float4* rp = reinterpret_cast<const float4*>(a.res32 + rbase + o0);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float4 q = __ldg(rp + j);
                f[4 * j] += q.x; f[4 * j + 1] += q.y; f[4 * j + 2] += q.z; f[4 * j + 3] += q.w;
              }
            } else {
              const uint4* rp = reinterpret_cast<const uint4*>(a.res + rbase + o0);
              const uint4 r0 = __ldg(rp), r1 = __ldg(rp + 1);
              const uint32_t u[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                f[2 * j] += __uint_as_float(u[j] << 16);
                f[2 * j + 1] += __uint_as_float(u[j] & 0xFFFF0000u);
              }
            }
          } else if (a.res_mode == 2) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int ci = o0 + j - a.r_pad_lo;
              if (ci >= 0 && ci < a.rC)
                f[j] += a.res32 ? __ldg(a.res32 + rbase + ci) : __uint_as_float((uint32_t)a.res[rbase + ci] << 16);
            }
          }
          if (a.relu) {
#pragma unroll
            for (int j = 0; j < 16; ++j) f[j] = fmaxf(f[j], 0.0f);
          }
          uint4 o0v, o1v;
          o0v.x = pack_bf16x2(f[0], f[1]);
          o0v.y = pack_bf16x2(f[2], f[3]);
          o0v.z = pack_bf16x2(f[4], f[5]);
          o0v.w = pack_bf16x2(f[6], f[7]);
          o1v.x = pack_bf16x2(f[8], f[9]);
          o1v.y = pack_bf16x2(f[10], f[11]);
          o1v.z = pack_bf16x2(f[12], f[13]);
          o1v.w = pack_bf16x2(f[14], f[15]);
          uint4* yp = reinterpret_cast<uint4*>(a.y + m * a.Cout + o0);
          yp[0] = o0v;
          yp[1] = o1v;
          if (a.y32) {
            float4* yq = reinterpret_cast<float4*>(a.y32 + m * a.Cout + o0);
#pragma unroll
            for (int j = 0; j < 4; ++j) yq[j] = make_float4(f[4 * j], f[4 * j + 1], f[4 * j + 2], f[4 * j + 3]);
          }
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(tempty0 + 8 * acc);
    }
  }

  __syncthreads();
  if (warp == 5) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
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

bool plan_geom(const ConvArgs& a, int BN, TmaGeom* g, int* stages, int* tiles_per_group) {
  if (a.Wo * a.stride > 256 || a.Wo > BM) return false;
  if (a.C == 8 || a.C == 16 || a.C == 32 || a.C == 64) g->CW = a.C;
  else if (a.C % 64 == 0) g->CW = 64;
  else return false;
  g->cchunks = a.C / g->CW;
  g->row_bytes = g->CW * 2;
  g->layout = g->row_bytes == 16 ? 0 : g->row_bytes == 32 ? 6 : g->row_bytes == 64 ? 4 : 2;
  g->nunits = a.ksz * a.ksz * g->cchunks;
  if (g->CW == 8 && (g->nunits & 1)) g->nunits += 1;       // pair units into 16-element K steps
  if (g->nunits * g->CW > a.Kp) return false;
  g->unit_bytes = BM * g->row_bytes;
  g->b_unit_bytes = BN * g->row_bytes;
  const int HoWo = a.Ho * a.Wo;
  if (HoWo >= BM) {
    g->bn = 1;
    g->bh = BM / a.Wo;
    if (g->bh > a.Ho) g->bh = a.Ho;
    *tiles_per_group = (a.Ho + g->bh - 1) / g->bh;
  } else {
    g->bh = a.Ho;
    g->bn = BM / HoWo;
    if (g->bn > 256) g->bn = 256;
    *tiles_per_group = 1;
  }
  if (g->bh * a.stride > 256) return false;
  g->rows = g->bn * g->bh * a.Wo;
  const int n_tiles = a.Cout / BN;
  const int b_total = (g->nunits * g->b_unit_bytes * n_tiles + 1023) & ~1023;
  const int avail = SMEM_BUDGET - b_total - 512;
  // units per stage: up to ~48 KB of A per stage, at least 3 stages in the ring
  int U = (48 * 1024) / g->unit_bytes;
  if (U > g->nunits) U = g->nunits;
  if (g->CW == 8 && (U & 1)) U -= 1;
  if (U < 1) U = 1;
  while (U > (g->CW == 8 ? 2 : 1) && avail / (U * g->unit_bytes) < 3) U -= (g->CW == 8 ? 2 : 1);
  g->U = U;
  g->nks = (g->nunits + U - 1) / U;
  int s = avail / (U * g->unit_bytes);
  if (s > 8) s = 8;
  if (s < 2) return false;
  *stages = s;
  return true;
}

template <int BN>
cudaError_t launch_tma_bn(const ConvArgs& a, int max_rows, int num_sms, cudaStream_t stream, bool* handled) {
  TmaParams P;
  P.a = a;
  if (!plan_geom(a, BN, &P.g, &P.stages, &P.tiles_per_img_group)) {
    *handled = false;
    return cudaSuccess;
  }
  EncodeTiledFn enc = get_encode();
  if (!enc) {
    *handled = false;
    return cudaSuccess;
  }
  const TmaGeom& G = P.g;
  CUtensorMap tmA, tmB;
  {
    const int n_alloc = max_rows + G.bn;     // rows a tile may touch (the buffer holds >= max_rows)
    (void)n_alloc;
    cuuint64_t dims[4] = {(cuuint64_t)a.C, (cuuint64_t)a.W, (cuuint64_t)a.H, (cuuint64_t)max_rows};
    cuuint64_t strides[3] = {(cuuint64_t)a.C * 2, (cuuint64_t)a.W * a.C * 2, (cuuint64_t)a.H * a.W * a.C * 2};
    cuuint32_t box[4] = {(cuuint32_t)G.CW, (cuuint32_t)(a.Wo * a.stride), (cuuint32_t)(G.bh * a.stride),
                         (cuuint32_t)G.bn};
    cuuint32_t es[4] = {1, (cuuint32_t)a.stride, (cuuint32_t)a.stride, 1};
    const CUtensorMapSwizzle sw = G.layout == 0 ? CU_TENSOR_MAP_SWIZZLE_NONE
                                  : G.layout == 6 ? CU_TENSOR_MAP_SWIZZLE_32B
                                  : G.layout == 4 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
    CUresult r = enc(&tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, (void*)a.x, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    cuuint64_t wd[2] = {(cuuint64_t)a.Kp, (cuuint64_t)a.Cout};
    cuuint64_t ws[1] = {(cuuint64_t)a.Kp * 2};
    cuuint32_t wb[2] = {(cuuint32_t)G.CW, (cuuint32_t)BN};
    cuuint32_t we[2] = {1, 1};
    r = enc(&tmB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void*)a.w, wd, ws, wb, we, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  }
  const int n_tiles = a.Cout / BN;
  const int b_total = (G.nunits * G.b_unit_bytes * n_tiles + 1023) & ~1023;
  const int smem = 1024 + b_total + P.stages * G.U * G.unit_bytes + 256;
  static int attr = 0;
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(k_conv_tma<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BUDGET + 2048);
    if (e != cudaSuccess) return e;
    attr = SMEM_BUDGET + 2048;
  }
  const long long groups = (max_rows + G.bn - 1) / G.bn;
  const long long tiles = groups * P.tiles_per_img_group * n_tiles;
  int grid = (int)(tiles < num_sms ? tiles : num_sms);
  if (grid < 1) grid = 1;
  *handled = true;
  k_conv_tma<BN><<<grid, THREADS, smem, stream>>>(tmA, tmB, P);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_conv_tma(const ConvArgs& a, int max_rows, int num_sms, cudaStream_t stream, bool* handled) {
  *handled = false;
  switch (a.Cout) {
    case 16: return launch_tma_bn<16>(a, max_rows, num_sms, stream, handled);
    case 32: return launch_tma_bn<32>(a, max_rows, num_sms, stream, handled);
    case 64: return launch_tma_bn<64>(a, max_rows, num_sms, stream, handled);
    case 128: return launch_tma_bn<128>(a, max_rows, num_sms, stream, handled);
    case 256: return launch_tma_bn<256>(a, max_rows, num_sms, stream, handled);
    default: return cudaSuccess;
  }
}

cudaError_t launch_conv(const ConvArgs& a, int max_rows, int num_sms, cudaStream_t stream, int path) {
  if (path != 1) {
    bool handled = false;
    cudaError_t e = launch_conv_tma(a, max_rows, num_sms, stream, &handled);
    if (e != cudaSuccess || handled) return e;
    if (path == 2) return cudaErrorNotSupported;
  }
  return launch_conv_tc(a, max_rows, num_sms, stream);
}

}  // namespace dycl
