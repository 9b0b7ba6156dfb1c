// NHWC implicit-GEMM convolution on tcgen05 with TMA im2col operand loads (SURVEY §8(a) a1,
// the ImageNet-scale layers of config 5: 1x1 / 3x3 / strided convs with C_in, C_out >= 64).
//
//   D[m, o] = sum_{r,s,c} X[n, ho*st - pad + r, wo*st - pad + s, c] * W[o, (r*k + s)*C + c]
//   m = flat output pixel (n, ho, wo) -- M runs across samples, so a 128-row tile never
//   wastes rows on a sample boundary (7x7 maps at stage 4 would waste 62% with per-sample
//   tiles).
//
// A operand (activations, bf16 NHWC [n][H][W][C]): one TMA im2col box per (tap, 64-channel
// block): 128 consecutive output pixels x 64 channels, the tap given as the im2col offset,
// the conv's zero padding and stride done by the TMA unit (bounding box = the output grid,
// traversal stride = conv stride; verified in tools/im2col_probe.cu).  1x1 / stride-1 layers
// use a plain 2-D tiled box of the [M][C] matrix.  B operand (weights [Cout][k*k*C], K
// ordered (r, s, c)): a 2-D tiled box.  Both land in SMEM in the 128-byte-swizzled K-major
// layout; tcgen05.mma 128 x BN x 16 reads them by descriptor.
//
// Persistent warp-specialised CTA (one per SM): warps 8, 10, 11 = TMA producers (k-blocks round-robin), warp 9 =
// TMEM allocator + MMA issuer (one lane), warps 0-7 = two epilogue warpgroups alternating
// tiles over two TMEM accumulators.  The fused epilogue adds bias (+ identity shortcut from
// the fp32 residual stream or the bf16 tensor), applies ReLU and writes bf16 NHWC (+ the fp32
// stream copy).  Tiles are numbered with the N tile fastest, so the CTAs running at the same
// time share A tiles through L2.
#include <cuda.h>
#include <cuda_bf16.h>

#include "kernels.h"
#include "ptx.cuh"

namespace dycl {
namespace {


constexpr int BM = 128;
constexpr int BKE = 64;                 // K elements per stage: one 128-byte swizzle row
constexpr int THREADS = 384;   // warps 0-7 epilogue, 8/10/11 TMA producers, 9 MMA
constexpr int NPROD = 3;

template <int BN>
struct CG {
  static constexpr int A_BYTES = BM * BKE * 2;
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
};
constexpr int MAX_STAGES = 8;
constexpr int SMEM_LIMIT = 227 * 1024;
constexpr int SMEM_MISC = 1024 + 512;        // alignment slack + barriers
// TMA-staged epilogue, per warpgroup: residual chunk (128 rows x 32 fp32, SW128), fp32 output
// chunk (SW128) and bf16 output chunk (128 rows x 32 bf16 = 64 B, SW64).
constexpr int EPI_RES = BM * 32 * 4, EPI_O32 = BM * 32 * 4, EPI_O16 = BM * 32 * 2;
constexpr int EPI_WG = EPI_RES + EPI_O32 + EPI_O16;

struct GemmPlan {
  int stages;      // mainloop ring depth
  int staged;      // 1: epilogue through SMEM + TMA stores (and TMA residual loads)
  int bres;        // 1: all weights resident in SMEM (single N tile, loaded once per CTA); the
                   //    ring then carries only A tiles (cuts L2->SMEM bytes by B/(A+B) per tile)
  int tshift;      // 1: stride-1 'same' conv whose whole samples tile BM: tap (r, s) of the A tile is
                   //    one TILED 4-d box {BKE, W, H, samples} at (c, s - pad, r - pad, n0) with zero
                   //    out-of-bounds fill -- same SMEM image as the im2col box, far fewer TMA requests
  int g1;          // zero-copy entry: rows per A box (the largest power of two <= 64 dividing HW)
  int g2;          // zero-copy entry: pixels per projection im2col box (largest power of two <= 16
                   //    dividing Ho*Wo); a box never straddles two samples
};

__device__ __forceinline__ void tma_im2col_4d(uint32_t dst, const void* tmap, uint32_t bar, int c, int w, int h, int n,
                                              uint16_t ow, uint16_t oh) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
      "%6}], [%2], {%7, %8};" ::"r"(dst),
      "l"(tmap), "r"(bar), "r"(c), "r"(w), "r"(h), "r"(n), "h"(ow), "h"(oh)
      : "memory");
}

__device__ __forceinline__ void ts_mark(const ConvArgs& a, int k) {   // development timeline
  if (a.ts && blockIdx.x < 8) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.ts[blockIdx.x * 16 + k] = (long long)t;
  }
}
__device__ __forceinline__ uint32_t pk2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
// the lo halves of the pair stream: bf16_rn(v - bf16_rn(v)) for two values
__device__ __forceinline__ uint32_t pk2lo(float a, float b) {
  const uint32_t h = pk2(a, b);
  return pk2(a - __uint_as_float(h << 16), b - __uint_as_float(h & 0xFFFF0000u));
}
__device__ __forceinline__ void wg_sync(int wg) { asm volatile("bar.sync %0, 128;" ::"r"(1 + wg) : "memory"); }
// 16-byte chunk j of row r in a 1024-B-aligned buffer with 128-byte rows, 128B swizzle
__device__ __forceinline__ uint32_t sw128(int r, int j) { return (uint32_t)(r * 128 + ((j ^ (r & 7)) << 4)); }
// 16-byte chunk j of row r with 64-byte rows, 64B swizzle (chunk bits XOR address bits [7,9))
__device__ __forceinline__ uint32_t sw64(int r, int j) { return (uint32_t)(r * 64 + ((j ^ ((r >> 1) & 3)) << 4)); }

// RT ("row-tap"): 3x3 / stride-1 'same' conv on whole-sample tiles (GemmPlan::tshift) with
// the three horizontal taps stacked along N (weights pack_rowtap, N = 3 * BN) and only the
// three vertical taps along K: a third of the A-operand traffic; the epilogue combines
// out(x) = T0(x-1) + T1(x) + T2(x+1) with lane shuffles (image rows never straddle a warp).
template <int BN, bool IM2COL, bool RT = false>
__global__ void __launch_bounds__(THREADS, 1)
    k_conv_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmR, const __grid_constant__ CUtensorMap tmY32,
                const __grid_constant__ CUtensorMap tmY16, const __grid_constant__ CUtensorMap tmA2,
                const __grid_constant__ CUtensorMap tmAL, const __grid_constant__ CUtensorMap tmRL,
                const ConvArgs a, const GemmPlan pl) {
  using G = CG<BN>;
  constexpr int NA = RT ? 3 * BN : BN;                     // MMA N = accumulator columns per tile
  constexpr int BB = NA * BKE * 2;                         // B bytes per k-block
  constexpr int TCOLS = RT ? 512 : G::TMEM_COLS;
  const int S = pl.stages;
  const int kblocks1 = (RT ? a.ksz : a.ksz * a.ksz) * (a.C / BKE);
  const int kblocks = kblocks1 + (a.x2 ? a.C2 / BKE : 0);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * G::A_BYTES;                     // ring B tiles, or [kblocks][BN][128 B] resident
  const int b_slots = pl.bres ? kblocks : S;
  uint8_t* sE = sB + b_slots * BB;                  // [2 WG][res | o32 | o16] when staged
  uint64_t* bars = reinterpret_cast<uint64_t*>(sE + (pl.staged ? 2 * EPI_WG : 0));
  const uint32_t full0 = ptx::smem_u32(bars);
  const uint32_t empty0 = full0 + 8 * S;
  const uint32_t tfull0 = empty0 + 8 * S;
  const uint32_t tempty0 = tfull0 + 16;
  const uint32_t rbar0 = tempty0 + 16;
  const uint32_t bfull = rbar0 + 16;                       // resident weights landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 7);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_live = a.n_live ? *a.n_live : a.n_static;
  // loop-invariant arguments laundered into registers: the asm "memory" clobbers in the
  // pipeline loops otherwise make the compiler re-read them from the parameter bank on every
  // iteration (constant-cache latency on the producer / MMA critical path)
  auto reg = [](int v) {
    int r;
    asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
    return r;
  };
  const int dbg = reg(a.dbg), pad = reg(a.pad), cstride = reg(a.stride), Wo = reg(a.Wo), ksz = reg(a.ksz);
  const int stride2 = reg(a.stride2);
  const int* const rows_in = reinterpret_cast<const int*>(
      (uintptr_t)(((unsigned long long)reg((int)((uintptr_t)a.rows_in >> 32)) << 32) |
                  (unsigned)reg((int)(uintptr_t)a.rows_in)));
  const int HWo = a.Ho * a.Wo;
  const long long M = (long long)n_live * HWo;
  const int m_tiles = (int)((M + BM - 1) / BM);
  const int n_tiles = a.Cout / BN;
  const int num_tiles = m_tiles * n_tiles;
  const int cblocks = a.C / BKE;

  if (threadIdx.x == 0) {
    ts_mark(a, 0);
    for (int i = 0; i < S; ++i) {
      ptx::mbar_init(full0 + 8 * i, 1);
      ptx::mbar_init(empty0 + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(tfull0 + 8 * i, 1);
      ptx::mbar_init(tempty0 + 8 * i, 128);
      ptx::mbar_init(rbar0 + 8 * i, 1);
    }
    ptx::mbar_init(bfull, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 9) ptx::tmem_alloc(ptx::smem_u32(tmem_slot), TCOLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) ts_mark(a, 1);

  if (warp == 8 || warp >= 10) {
    // ------------------------------------------------------------ TMA producers
    // A single issuing warp runs at ~9 cycles per instruction (one dependent stream), i.e.
    // ~400-600 cycles per k-block -- slower than the tensor core eats a 128x64x64 block
    // (measured with a globaltimer timeline).  NPROD warps on different SM sub-partitions take
    // the k-blocks round-robin; each walks the whole loop (waits by all lanes, issue by lane 0).
    const int prod = warp == 8 ? 0 : warp - 9;
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tmA);
      ptx::tma_prefetch_desc(&tmB);
      if (a.x2) ptx::tma_prefetch_desc(&tmA2);
      if (pl.bres && prod == 0) {
        ptx::mbar_arrive_expect_tx(bfull, (uint32_t)(kblocks * BB));
        for (int kb = 0; kb < kblocks; ++kb)
          ptx::tma_load_2d(ptx::smem_u32(sB + kb * BB), &tmB, bfull, kb * BKE, 0);
      }
    }
    __syncwarp();
    const uint32_t stage_tx = pl.bres ? (uint32_t)G::A_BYTES : (uint32_t)(G::A_BYTES + BB);
    // this producer's k-blocks: global sequence numbers prod, prod + NPROD, ...
    // at most S producers: a producer then never runs two ring rounds ahead of a stage's
    // empty barrier, which a parity wait could not tell apart
    const int np = NPROD < S ? NPROD : S;
    int stage = prod;
    uint32_t phase = 0;
    int rr = 0;                                    // round-robin owner of the next k-block
    auto advance = [&]() {
      stage += np;
      while (stage >= S) {
        stage -= S;
        phase ^= 1;
      }
    };
    for (int tile = blockIdx.x; tile < (prod >= np ? 0 : num_tiles); tile += gridDim.x) {
      if (lane == 0 && prod == 0 && tile == (int)blockIdx.x + (int)gridDim.x) ts_mark(a, 5);
      const int m_tile = tile / n_tiles, n_tile = tile - m_tile * n_tiles;
      const long long p0 = (long long)m_tile * BM;
      const int n0 = (int)(p0 / HWo);
      const int rem = (int)(p0 - (long long)n0 * HWo);
      const int ho0 = rem / Wo, wo0 = rem - (rem / Wo) * Wo;
      const int wb = wo0 * cstride - pad, hb = ho0 * cstride - pad;
      int kb = 0;
      for (int r = 0; r < ksz; ++r)
        for (int s = RT ? 1 : 0; s < (RT ? 2 : ksz); ++s)
          for (int cb = 0; cb < cblocks; ++cb, ++kb) {
            const bool mine = rr == prod;
            rr = rr + 1 == np ? 0 : rr + 1;
            if (!mine) continue;
            ptx::mbar_wait(empty0 + 8 * stage, phase ^ 1);
            if (lane == 0) {
              const uint32_t bar = full0 + 8 * stage;
              const uint32_t da = ptx::smem_u32(sA + stage * G::A_BYTES);
              if (dbg & 1024) {                    // timing experiment: no operand loads
                ptx::mbar_arrive(bar);
              } else {
                ptx::mbar_arrive_expect_tx(bar, stage_tx);
                if (IM2COL && rows_in) {
                  // whole-sample tiles through the row list: one HWo-pixel box per sample
                  const int spt = BM / HWo;
                  for (int sp = 0; sp < spt; ++sp) {
                    const int idx = m_tile * spt + sp;
                    const int nn = rows_in[idx < n_live ? idx : 0];
                    if (pl.tshift)
                      ptx::tma_load_4d(da + (uint32_t)(sp * HWo * BKE * 2), &tmAL, bar, cb * BKE, s - pad,
                                       r - pad, nn);
                    else
                      tma_im2col_4d(da + (uint32_t)(sp * HWo * BKE * 2), &tmAL, bar, cb * BKE, -pad, -pad, nn,
                                    (uint16_t)s, (uint16_t)r);
                  }
                } else if (!IM2COL && a.rows_gather) {
                  // zero-copy entry: BM / g1 boxes of g1 rows, each inside one input sample
                  // (1x1 / stride 1: HW == HWo; sample and pixel advanced incrementally, no divisions)
                  int idx = n0, prow = rem;
                  for (int h = 0; h < BM / pl.g1; ++h) {
                    const int src = a.rows_gather[idx < n_live ? idx : (n_live > 0 ? n_live - 1 : 0)];
                    ptx::tma_load_3d(da + (uint32_t)(h * pl.g1 * BKE * 2), &tmAL, bar, cb * BKE, prow, src);
                    prow += pl.g1;
                    if (prow >= HWo) {
                      prow -= HWo;
                      ++idx;
                    }
                  }
                } else if (IM2COL && pl.tshift) {
                  ptx::tma_load_4d(da, &tmA, bar, cb * BKE, s - pad, r - pad, n0);
                } else if (IM2COL) {
                  tma_im2col_4d(da, &tmA, bar, cb * BKE, wb, hb, n0, (uint16_t)s, (uint16_t)r);
                } else {
                  ptx::tma_load_2d(da, &tmA, bar, cb * BKE, (int)p0);
                }
                if (!pl.bres)
                  ptx::tma_load_2d(ptx::smem_u32(sB + stage * BB), &tmB, bar, kb * BKE, n_tile * NA);
              }
            }
            __syncwarp();
            advance();
          }
      // fused projection shortcut: K blocks of the second operand (1x1, stride2)
      for (int cb = 0; kb < kblocks; ++cb, ++kb) {
        const bool mine = rr == prod;
        rr = rr + 1 == np ? 0 : rr + 1;
        if (!mine) continue;
        ptx::mbar_wait(empty0 + 8 * stage, phase ^ 1);
        if (lane == 0) {
          const uint32_t bar = full0 + 8 * stage;
          ptx::mbar_arrive_expect_tx(bar, stage_tx);
          const uint32_t da = ptx::smem_u32(sA + stage * G::A_BYTES);
          if (a.x2_rows) {
            // zero-copy entry: BM / g2 im2col boxes of g2 pixels, each inside one sample; the
            // (sample, output row, output column) of each box advanced incrementally, no divisions
            int idx = n0, ho = ho0, wo = wo0;
            for (int q = 0; q < BM / pl.g2; ++q) {
              const int src = a.x2_rows[idx < n_live ? idx : (n_live > 0 ? n_live - 1 : 0)];
              tma_im2col_4d(da + (uint32_t)(q * pl.g2 * BKE * 2), &tmA2, bar, cb * BKE, wo * stride2, ho * stride2,
                            src, 0, 0);
              wo += pl.g2;
              while (wo >= Wo) {
                wo -= Wo;
                if (++ho == a.Ho) {
                  ho = 0;
                  ++idx;
                }
              }
            }
          } else if (stride2 > 1)
            tma_im2col_4d(da, &tmA2, bar, cb * BKE, wo0 * stride2, ho0 * stride2, n0, 0, 0);
          else
            ptx::tma_load_2d(da, &tmA2, bar, cb * BKE, (int)p0);
          if (!pl.bres)
            ptx::tma_load_2d(ptx::smem_u32(sB + stage * BB), &tmB, bar, kb * BKE, n_tile * NA);
        }
        __syncwarp();
        advance();
      }
    }
    if (lane == 0 && prod == 0) ts_mark(a, 6);
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t IDESC = ptx::make_idesc_bf16(BM, NA);
    if (pl.bres) ptx::mbar_wait(bfull, 0);
    if (lane == 0) ts_mark(a, 2);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      ptx::mbar_wait(tempty0 + 8 * acc, ((it >> 1) & 1) ^ 1);
      ptx::tc_fence_after();
      const uint32_t d = tmem_base + (uint32_t)(acc * NA);
      for (int kb = 0; kb < kblocks; ++kb) {
        ptx::mbar_wait(full0 + 8 * stage, phase);
        ptx::tc_fence_after();
        const uint64_t ad = ptx::make_smem_desc_sw128(ptx::smem_u32(sA + stage * G::A_BYTES));
        const uint64_t bd = ptx::make_smem_desc_sw128(ptx::smem_u32(sB + (pl.bres ? kb : stage) * BB));
        if (ptx::elect_one() && !(dbg & 2048)) {   // dbg 2048: timing experiment, no MMAs
#pragma unroll
          for (int j = 0; j < BKE / 16; ++j)
            ptx::mma_bf16_ss_lohi(d, (uint32_t)ad + 2 * j, (uint32_t)(ad >> 32), (uint32_t)bd + 2 * j,
                                  (uint32_t)(bd >> 32), IDESC, (uint32_t)((kb | j) != 0));
        }
        __syncwarp();
        ptx::mma_commit_elect(empty0 + 8 * stage);
        __syncwarp();
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
      ptx::mma_commit_elect(tfull0 + 8 * acc);
      __syncwarp();
      if (lane == 0 && it == 0) ts_mark(a, 3);
    }
    if (lane == 0) {
      ts_mark(a, 4);
      if (a.ts && blockIdx.x < 8) a.ts[blockIdx.x * 16 + 10] = it;
    }
  } else {
    // ------------------------------------------------------------ epilogue (2 warpgroups)
    const int wg = warp >> 2, quad = warp & 3;
    const int r = quad * 32 + lane;                         // TMEM lane = row of the tile
    const bool leader = (threadIdx.x & 127) == 0;
    const bool res = a.res_mode == 1;
    const bool res_f = res && a.res32 != nullptr;
    // pair stream (ConvArgs::y32_pair): the residual stream is bf16 hi (the operand copy a.res /
    // a.y) + bf16 lo (the planes behind res32 / y32), value = hi + lo
    const bool pair = a.y32_pair != 0;
    const uint16_t* res_lo = reinterpret_cast<const uint16_t*>(a.res32);
    uint16_t* y_lo = reinterpret_cast<uint16_t*>(a.y32);
    const bool staged = pl.staged != 0;
    uint8_t* eR = sE + wg * EPI_WG;
    uint8_t* eO32 = eR + EPI_RES;
    uint8_t* eO16 = eO32 + EPI_O32;
    const uint32_t rbar = rbar0 + 8 * wg;
    uint32_t rphase = 0;
    if (staged && leader) {
      if (res) ptx::tma_prefetch_desc(&tmR);
      if (a.y32) ptx::tma_prefetch_desc(&tmY32);
      if (res_f && pair) ptx::tma_prefetch_desc(&tmRL);
      if (a.y) ptx::tma_prefetch_desc(&tmY16);
    }
    int it = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      if ((it & 1) != wg) continue;
      const int acc = it & 1;
      if (a.dbg & 4096) {                            // timing experiment: no epilogue work
        ptx::mbar_wait(tfull0 + 8 * acc, (it >> 1) & 1);
        ptx::tc_fence_after();
        ptx::tc_fence_before();
        ptx::mbar_arrive(tempty0 + 8 * acc);
        continue;
      }
      const int m_tile = tile / n_tiles, n_tile = tile - m_tile * n_tiles;
      const long long m0 = (long long)m_tile * BM;
      const long long m = m0 + r;
      bool ok = m < M;
      const bool full = m0 + BM <= M;
      const int col0 = n_tile * BN;
      long long mo = m;                                       // output row (list mode: remapped)
      if (a.rows_in || a.rows_out) {
        const int spt = BM / HWo;
        const int idx = m_tile * spt + r / HWo;
        ok = idx < n_live;
        mo = (long long)(a.rows_out && ok ? a.rows_out[idx] : idx) * HWo + r % HWo;
      }
      const size_t rowo = (size_t)(ok ? mo : 0) * a.Cout + col0;
      auto res_load = [&](int c0) {
        ptx::mbar_arrive_expect_tx(rbar, res_f ? EPI_RES : EPI_RES / 2);
        ptx::tma_load_2d(ptx::smem_u32(eR), &tmR, rbar, col0 + c0, (int)m0);
        if (res_f && pair) ptx::tma_load_2d(ptx::smem_u32(eR + EPI_RES / 2), &tmRL, rbar, col0 + c0, (int)m0);
      };
      if (staged && res && leader) res_load(0);
      // unstaged shortcut chunk (32 channels) prefetch, issued before the accumulator wait
      float4 rs[8];
      auto load_res_g = [&](int c0) {
        if (res_f && pair) {
          const uint4* qh = reinterpret_cast<const uint4*>(a.res + rowo + c0);
          const uint4* ql = reinterpret_cast<const uint4*>(res_lo + rowo + c0);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint4 h = ok ? __ldg(qh + j) : make_uint4(0, 0, 0, 0);
            const uint4 l = ok ? __ldg(ql + j) : make_uint4(0, 0, 0, 0);
            rs[2 * j] = make_float4(__uint_as_float(h.x << 16) + __uint_as_float(l.x << 16),
                                    __uint_as_float(h.x & 0xFFFF0000u) + __uint_as_float(l.x & 0xFFFF0000u),
                                    __uint_as_float(h.y << 16) + __uint_as_float(l.y << 16),
                                    __uint_as_float(h.y & 0xFFFF0000u) + __uint_as_float(l.y & 0xFFFF0000u));
            rs[2 * j + 1] = make_float4(__uint_as_float(h.z << 16) + __uint_as_float(l.z << 16),
                                        __uint_as_float(h.z & 0xFFFF0000u) + __uint_as_float(l.z & 0xFFFF0000u),
                                        __uint_as_float(h.w << 16) + __uint_as_float(l.w << 16),
                                        __uint_as_float(h.w & 0xFFFF0000u) + __uint_as_float(l.w & 0xFFFF0000u));
          }
        } else if (res_f) {
          const float4* q = reinterpret_cast<const float4*>(a.res32 + rowo + c0);
#pragma unroll
          for (int j = 0; j < 8; ++j) rs[j] = ok ? __ldg(q + j) : make_float4(0.f, 0.f, 0.f, 0.f);
        } else if (res) {
          const uint4* q = reinterpret_cast<const uint4*>(a.res + rowo + c0);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint4 u = ok ? __ldg(q + j) : make_uint4(0, 0, 0, 0);
            rs[2 * j] = make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u),
                                    __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xFFFF0000u));
            rs[2 * j + 1] = make_float4(__uint_as_float(u.z << 16), __uint_as_float(u.z & 0xFFFF0000u),
                                        __uint_as_float(u.w << 16), __uint_as_float(u.w & 0xFFFF0000u));
          }
        }
      };
      if (!staged && res) load_res_g(0);
      ptx::mbar_wait(tfull0 + 8 * acc, (it >> 1) & 1);
      ptx::tc_fence_after();
      const uint32_t t_base = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * NA);
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t v[32];
        if constexpr (RT) {
          // out(x) = T0(x-1) + T1(x) + T2(x+1); x = tile row mod W (whole samples per tile)
          const int xr = r % Wo;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t t0[16], t2[16];
            ptx::tmem_ld_32x32b_x16(t_base + (uint32_t)(c0 + 16 * h), t0);
            ptx::tmem_ld_32x32b_x16(t_base + (uint32_t)(BN + c0 + 16 * h), *reinterpret_cast<uint32_t(*)[16]>(v + 16 * h));
            ptx::tmem_ld_32x32b_x16(t_base + (uint32_t)(2 * BN + c0 + 16 * h), t2);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float lft = __shfl_up_sync(0xffffffffu, __uint_as_float(t0[j]), 1);
              const float rgt = __shfl_down_sync(0xffffffffu, __uint_as_float(t2[j]), 1);
              float f = __uint_as_float(v[16 * h + j]);
              if (xr > 0) f += lft;
              if (xr < Wo - 1) f += rgt;
              v[16 * h + j] = __float_as_uint(f);
            }
          }
        } else {
          ptx::tmem_ld_32x32b_x16(t_base + (uint32_t)c0, *reinterpret_cast<uint32_t(*)[16]>(v));
          ptx::tmem_ld_32x32b_x16(t_base + (uint32_t)c0 + 16, *reinterpret_cast<uint32_t(*)[16]>(v + 16));
          ptx::tmem_ld_wait();
        }
        float f[32];
        {
          // bias as 8 broadcast 16-byte loads (col0 + c0 is a multiple of 32): the scalar form was
          // 32 loads per chunk, a fifth of the epilogue's instructions on the K = 64 convs
          const float4* b4 = reinterpret_cast<const float4*>(a.bias + col0 + c0);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 q = __ldg(b4 + j);
            f[4 * j] = __uint_as_float(v[4 * j]) + q.x;
            f[4 * j + 1] = __uint_as_float(v[4 * j + 1]) + q.y;
            f[4 * j + 2] = __uint_as_float(v[4 * j + 2]) + q.z;
            f[4 * j + 3] = __uint_as_float(v[4 * j + 3]) + q.w;
          }
        }
        if (staged && res) {
          ptx::mbar_wait(rbar, rphase);
          rphase ^= 1;
          if (res_f && pair) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint4 uh = *reinterpret_cast<const uint4*>(eR + sw64(r, j));
              const uint4 ul = *reinterpret_cast<const uint4*>(eR + EPI_RES / 2 + sw64(r, j));
              const uint32_t h4[4] = {uh.x, uh.y, uh.z, uh.w}, l4[4] = {ul.x, ul.y, ul.z, ul.w};
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                f[8 * j + 2 * q] += __uint_as_float(h4[q] << 16) + __uint_as_float(l4[q] << 16);
                f[8 * j + 2 * q + 1] += __uint_as_float(h4[q] & 0xFFFF0000u) + __uint_as_float(l4[q] & 0xFFFF0000u);
              }
            }
          } else if (res_f) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 q = *reinterpret_cast<const float4*>(eR + sw128(r, j));
              f[4 * j] += q.x; f[4 * j + 1] += q.y; f[4 * j + 2] += q.z; f[4 * j + 3] += q.w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint4 u = *reinterpret_cast<const uint4*>(eR + sw64(r, j));
              const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                f[8 * j + 2 * q] += __uint_as_float(w4[q] << 16);
                f[8 * j + 2 * q + 1] += __uint_as_float(w4[q] & 0xFFFF0000u);
              }
            }
          }
        } else if (res) {
          const float* rf = reinterpret_cast<const float*>(rs);
#pragma unroll
          for (int j = 0; j < 32; ++j) f[j] += rf[j];
          if (c0 + 32 < BN) load_res_g(c0 + 32);            // next chunk's shortcut in flight
        }
        if (a.res_mode == 2 && ok) {
          // option A: shortcut = block input pixel (2ho, 2wo), channel o - r_pad_lo, zero outside
          // [0, rC); r_pad_lo and rC are multiples of 4, so every 4-channel group is all in or out
          const long long nn = m / HWo;
          const int pp = (int)(m - nn * HWo), ho = pp / a.Wo, wo = pp - (pp / a.Wo) * a.Wo;
          const size_t rpix = (size_t)(2 * ho) * a.rW + 2 * wo;
#pragma unroll
          for (int g4 = 0; g4 < 8; ++g4) {
            const int ci = col0 + c0 + 4 * g4 - a.r_pad_lo;
            if (ci < 0 || ci + 4 > a.rC) continue;
            float4 q;
            if (a.res32) {
              q = __ldg(reinterpret_cast<const float4*>(a.res32 + ((size_t)nn * a.rH * a.rW + rpix) * a.rC + ci));
            } else {
              const uint16_t* rp = a.res_nhwc ? a.res + ((size_t)nn * a.rH * a.rW + rpix) * a.rC + ci
                                              : a.res + (size_t)nn * a.rC * a.rH * a.rW +
                                                    (size_t)(ci >> 3) * a.rH * a.rW * 8 + rpix * 8 + (ci & 7);
              const uint2 u = __ldg(reinterpret_cast<const uint2*>(rp));
              q = make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u),
                              __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xFFFF0000u));
            }
            f[4 * g4] += q.x; f[4 * g4 + 1] += q.y; f[4 * g4 + 2] += q.z; f[4 * g4 + 3] += q.w;
          }
        }
        if (a.relu) {
#pragma unroll
          for (int j = 0; j < 32; ++j) f[j] = fmaxf(f[j], 0.0f);
        }
        if (staged) {
          // all rows consumed the residual buffer; the previous chunk's stores have read the
          // output staging: refill the one, rewrite the other
          if (leader) ptx::bulk_wait_read0();
          wg_sync(wg);
          if (res && leader && c0 + 32 < BN) res_load(c0 + 32);
        }
        if (a.gap_part) {
          // fused GAP (a2): column sums of the chunk's fp32 y over groups of G consecutive rows
          // (G = the largest power of two <= 32 dividing HW: a group lies inside one sample and
          // covers the same pixels p in [kG, (k+1)G) whatever the sample's batch position) into
          // the partials [M / G][Cout]. A transpose-reduce over the warp's 32 rows (= lanes):
          // at level o = 1, 2, .., G/2 lanes l and l^o swap halves of their column sets and add,
          // so after log2(G) levels lane l holds 32/G column sums over its aligned G-row group --
          // a fixed pairwise tree (batch-position independent), no SMEM staging, no barrier
          const int G = a.gap_g;
          float g[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) g[j] = f[j];
          int colbase = 0;                                  // first column of this lane's set
#pragma unroll
          for (int lvl = 0; lvl < 5; ++lvl) {
            const int o = 1 << lvl;
            if (o >= G) break;
            const int n = 16 >> lvl;                         // columns kept after this level
            const bool upper = (lane & o) != 0;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              if (j < n) {
                const float send = upper ? g[j] : g[n + j];
                const float recv = __shfl_xor_sync(0xffffffffu, send, o);
                g[j] = (upper ? g[n + j] : g[j]) + recv;
              }
            }
            if (upper) colbase += n;
          }
          const int ncol = 32 / G;                           // column sums held by this lane
          const long long grow = m0 + 32 * quad + (lane & ~(G - 1));   // first row of the group
          if (grow < M) {
            float* gp = a.gap_part + (size_t)(grow / G) * a.Cout + col0 + c0 + colbase;
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (j < ncol) gp[j] = g[j];
          }
        }
        if (staged && full) {
          if (a.y32 && pair) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              *reinterpret_cast<uint4*>(eO32 + sw64(r, j)) =
                  make_uint4(pk2lo(f[8 * j], f[8 * j + 1]), pk2lo(f[8 * j + 2], f[8 * j + 3]),
                             pk2lo(f[8 * j + 4], f[8 * j + 5]), pk2lo(f[8 * j + 6], f[8 * j + 7]));
          } else if (a.y32) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              *reinterpret_cast<float4*>(eO32 + sw128(r, j)) = make_float4(f[4 * j], f[4 * j + 1], f[4 * j + 2], f[4 * j + 3]);
          }
          if (a.y) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              *reinterpret_cast<uint4*>(eO16 + sw64(r, j)) =
                  make_uint4(pk2(f[8 * j], f[8 * j + 1]), pk2(f[8 * j + 2], f[8 * j + 3]),
                             pk2(f[8 * j + 4], f[8 * j + 5]), pk2(f[8 * j + 6], f[8 * j + 7]));
          }
          ptx::fence_proxy_async_smem();
          wg_sync(wg);
          if (leader) {
            if (a.y32) ptx::tma_store_2d(&tmY32, ptx::smem_u32(eO32), col0 + c0, (int)m0);
            if (a.y) ptx::tma_store_2d(&tmY16, ptx::smem_u32(eO16), col0 + c0, (int)m0);
            ptx::bulk_commit();
          }
        } else if (ok) {
          if (a.y) {
            uint4* yq = reinterpret_cast<uint4*>(a.y + rowo + c0);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              yq[j] = make_uint4(pk2(f[8 * j], f[8 * j + 1]), pk2(f[8 * j + 2], f[8 * j + 3]),
                                 pk2(f[8 * j + 4], f[8 * j + 5]), pk2(f[8 * j + 6], f[8 * j + 7]));
          }
          if (a.y32 && pair) {
            uint4* lq = reinterpret_cast<uint4*>(y_lo + rowo + c0);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              lq[j] = make_uint4(pk2lo(f[8 * j], f[8 * j + 1]), pk2lo(f[8 * j + 2], f[8 * j + 3]),
                                 pk2lo(f[8 * j + 4], f[8 * j + 5]), pk2lo(f[8 * j + 6], f[8 * j + 7]));
          } else if (a.y32) {
            float4* zq = reinterpret_cast<float4*>(a.y32 + rowo + c0);
#pragma unroll
            for (int j = 0; j < 8; ++j) zq[j] = make_float4(f[4 * j], f[4 * j + 1], f[4 * j + 2], f[4 * j + 3]);
          }
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(tempty0 + 8 * acc);
      if (threadIdx.x == 0 && it == 0) ts_mark(a, 7);
    }
    if (staged && leader) ptx::bulk_wait0();
    if (threadIdx.x == 0) ts_mark(a, 8);                 // stores done reading SMEM before exit
  }
  __syncthreads();
  if (threadIdx.x == 0) ts_mark(a, 9);
  if (warp == 9) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, TCOLS);
  }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
typedef CUresult (*EncodeIm2colFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t, const cuuint32_t*,
                                   CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill);

template <typename F>
F driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
    return reinterpret_cast<F>(p);
  return nullptr;
}

template <int BN, bool IM2COL, bool RT = false>
cudaError_t launch_t(const ConvArgs& a, int max_rows, int num_sms, cudaStream_t stream) {
  constexpr int NA = RT ? 3 * BN : BN;
  constexpr int BB = NA * BKE * 2;
  static EncodeTiledFn enc = driver_fn<EncodeTiledFn>("cuTensorMapEncodeTiled");
  static EncodeIm2colFn enc_i2c = driver_fn<EncodeIm2colFn>("cuTensorMapEncodeIm2col");
  if (!enc || !enc_i2c) return cudaErrorNotSupported;
  CUtensorMap tmA, tmB, tmR, tmY32, tmY16;
  const int rows = max_rows > 0 ? max_rows : 1;
  const cuuint64_t Mmax = (cuuint64_t)rows * a.Ho * a.Wo;
  if (IM2COL) {
    cuuint64_t dims[4] = {(cuuint64_t)a.C, (cuuint64_t)a.W, (cuuint64_t)a.H, (cuuint64_t)rows};
    cuuint64_t strides[3] = {(cuuint64_t)a.C * 2, (cuuint64_t)a.W * a.C * 2, (cuuint64_t)a.H * a.W * a.C * 2};
    // bounding box of the filter origins = the output grid: {W, H} order (tools/im2col_probe.cu)
    int lower[2] = {-a.pad, -a.pad};
    int upper[2] = {(a.Wo - 1) * a.stride - a.pad - (a.W - 1), (a.Ho - 1) * a.stride - a.pad - (a.H - 1)};
    cuuint32_t es[4] = {1, (cuuint32_t)a.stride, (cuuint32_t)a.stride, 1};
    if (enc_i2c(&tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, (void*)a.x, dims, strides, lower, upper, BKE, BM, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  } else {
    cuuint64_t dims[2] = {(cuuint64_t)a.C, (cuuint64_t)rows * a.H * a.W};
    cuuint64_t strides[1] = {(cuuint64_t)a.C * 2};
    cuuint32_t box[2] = {BKE, BM};
    cuuint32_t es[2] = {1, 1};
    if (enc(&tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void*)a.x, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  auto mat2d = [&](CUtensorMap* t, const void* p, CUtensorMapDataType dt, int esz, cuuint64_t inner, cuuint64_t outer,
                   cuuint32_t bi, cuuint32_t bo, CUtensorMapSwizzle sw) {
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {inner * (cuuint64_t)esz};
    cuuint32_t box[2] = {bi, bo};
    cuuint32_t es[2] = {1, 1};
    return enc(t, dt, 2, (void*)p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  if (RT ? !mat2d(&tmB, a.w_rt, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.Kp_rt, 3 * a.Cout, BKE, NA,
                  CU_TENSOR_MAP_SWIZZLE_128B)
         : !mat2d(&tmB, a.w, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.Kp, a.Cout, BKE, BN, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  CUtensorMap tmAL = tmB;
  if (IM2COL && a.rows_in) {
    cuuint64_t dims[4] = {(cuuint64_t)a.C, (cuuint64_t)a.W, (cuuint64_t)a.H, (cuuint64_t)rows};
    cuuint64_t strides[3] = {(cuuint64_t)a.C * 2, (cuuint64_t)a.W * a.C * 2, (cuuint64_t)a.H * a.W * a.C * 2};
    int lower[2] = {-a.pad, -a.pad};
    int upper[2] = {(a.Wo - 1) * a.stride - a.pad - (a.W - 1), (a.Ho - 1) * a.stride - a.pad - (a.H - 1)};
    cuuint32_t es[4] = {1, (cuuint32_t)a.stride, (cuuint32_t)a.stride, 1};
    if (enc_i2c(&tmAL, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, (void*)a.x, dims, strides, lower, upper, BKE,
                (cuuint32_t)(a.Ho * a.Wo), es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  const int g1 = zero_copy_rows(a.H * a.W, 64), g2 = zero_copy_rows(a.Ho * a.Wo, 16);
  if (!IM2COL && a.rows_gather) {
    if (g1 < ZC_MIN_ROWS) return cudaErrorInvalidValue;
    cuuint64_t dims[3] = {(cuuint64_t)a.C, (cuuint64_t)a.H * a.W, (cuuint64_t)rows};
    cuuint64_t strides[2] = {(cuuint64_t)a.C * 2, (cuuint64_t)a.H * a.W * a.C * 2};
    cuuint32_t box[3] = {BKE, (cuuint32_t)g1, 1};
    cuuint32_t es[3] = {1, 1, 1};
    if (enc(&tmAL, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, (void*)a.x, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  // tiled-shift A operand (GemmPlan::tshift)
  const int HW = a.H * a.W;
  const bool tshift = IM2COL && a.stride == 1 && a.Ho == a.H && a.Wo == a.W && 2 * a.pad + 1 == a.ksz && HW <= BM &&
                      BM % HW == 0 && !(a.dbg & 512);
  if (tshift) {
    cuuint64_t dims[4] = {(cuuint64_t)a.C, (cuuint64_t)a.W, (cuuint64_t)a.H, (cuuint64_t)rows};
    cuuint64_t strides[3] = {(cuuint64_t)a.C * 2, (cuuint64_t)a.W * a.C * 2, (cuuint64_t)a.H * a.W * a.C * 2};
    cuuint32_t es[4] = {1, 1, 1, 1};
    cuuint32_t box[4] = {BKE, (cuuint32_t)a.W, (cuuint32_t)a.H, (cuuint32_t)(BM / HW)};
    if (enc(&tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, (void*)a.x, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
    if (a.rows_in) {
      box[3] = 1;
      if (enc(&tmAL, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, (void*)a.x, dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    }
  }
  CUtensorMap tmA2 = tmB;
  if (a.x2 && a.x2_rows) {
    // g2-pixel strided im2col boxes of the projection operand (zero-copy entry)
    if (g2 < ZC_MIN_ROWS) return cudaErrorInvalidValue;
    cuuint64_t dims[4] = {(cuuint64_t)a.C2, (cuuint64_t)a.W2, (cuuint64_t)a.H2, (cuuint64_t)rows};
    cuuint64_t strides[3] = {(cuuint64_t)a.C2 * 2, (cuuint64_t)a.W2 * a.C2 * 2, (cuuint64_t)a.H2 * a.W2 * a.C2 * 2};
    int lower[2] = {0, 0};
    int upper[2] = {(a.Wo - 1) * a.stride2 - (a.W2 - 1), (a.Ho - 1) * a.stride2 - (a.H2 - 1)};
    cuuint32_t es[4] = {1, (cuuint32_t)a.stride2, (cuuint32_t)a.stride2, 1};
    if (enc_i2c(&tmA2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, (void*)a.x2, dims, strides, lower, upper, BKE, (cuuint32_t)g2, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  } else if (a.x2) {
    if (a.stride2 > 1) {
      cuuint64_t dims[4] = {(cuuint64_t)a.C2, (cuuint64_t)a.W2, (cuuint64_t)a.H2, (cuuint64_t)rows};
      cuuint64_t strides[3] = {(cuuint64_t)a.C2 * 2, (cuuint64_t)a.W2 * a.C2 * 2, (cuuint64_t)a.H2 * a.W2 * a.C2 * 2};
      int lower[2] = {0, 0};
      int upper[2] = {(a.Wo - 1) * a.stride2 - (a.W2 - 1), (a.Ho - 1) * a.stride2 - (a.H2 - 1)};
      cuuint32_t es[4] = {1, (cuuint32_t)a.stride2, (cuuint32_t)a.stride2, 1};
      if (enc_i2c(&tmA2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, (void*)a.x2, dims, strides, lower, upper, BKE, BM, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    } else if (!mat2d(&tmA2, a.x2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.C2, Mmax, BKE, BM,
                      CU_TENSOR_MAP_SWIZZLE_128B)) {
      return cudaErrorInvalidValue;
    }
  }
  // epilogue plan: SMEM-staged TMA stores when the epilogue moves more than a bf16 tile
  // (fp32 stream copy and / or a shortcut) and the ring keeps >= 2 stages beside the staging
  GemmPlan pl{};
  pl.tshift = tshift;
  pl.g1 = g1;
  pl.g2 = g2;
  if (RT && !tshift) return cudaErrorInvalidValue;
  const int kblocks = (RT ? a.ksz : a.ksz * a.ksz) * (a.C / BKE) + (a.x2 ? a.C2 / BKE : 0);
  const bool heavy = a.y32 != nullptr || a.res_mode == 1;
  const int avail_staged = SMEM_LIMIT - SMEM_MISC - 2 * EPI_WG;
  pl.staged = (heavy || a.gap_part) && avail_staged / (CG<BN>::A_BYTES + BB) >= 2 && !(a.dbg & 128) && !a.rows_out &&
              !a.rows_in;
  if (a.gap_part && !pl.staged) return cudaErrorNotSupported;   // (the fused GAP is planned with the staged epilogue)
  const int avail = pl.staged ? avail_staged : SMEM_LIMIT - SMEM_MISC;
  // resident weights: one N tile whose K blocks all fit beside >= 3 A stages
  pl.bres = a.Cout == BN && kblocks > 1 && avail - kblocks * BB >= 3 * CG<BN>::A_BYTES && !(a.dbg & 256);
  pl.stages = pl.bres ? (avail - kblocks * BB) / CG<BN>::A_BYTES : avail / (CG<BN>::A_BYTES + BB);
  if (pl.stages > MAX_STAGES) pl.stages = MAX_STAGES;
  if (pl.stages > kblocks + 1 && kblocks >= 1) pl.stages = kblocks + 1 > 2 ? kblocks + 1 : 2;
  CUtensorMap tmRL = tmB;
  tmR = tmY32 = tmY16 = tmB;
  const bool pair = a.y32_pair != 0;
  if (pair && a.res_mode == 1 && a.res32 && !a.res) return cudaErrorInvalidValue;   // the hi plane
  if (pl.staged) {
    if (a.res_mode == 1 && a.res32 && pair) {
      if (!mat2d(&tmR, a.res, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.Cout, Mmax, 32, BM, CU_TENSOR_MAP_SWIZZLE_64B) ||
          !mat2d(&tmRL, a.res32, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.Cout, Mmax, 32, BM, CU_TENSOR_MAP_SWIZZLE_64B))
        return cudaErrorInvalidValue;
    } else if (a.res_mode == 1) {
      const bool f32 = a.res32 != nullptr;
      if (!mat2d(&tmR, f32 ? (const void*)a.res32 : (const void*)a.res,
                 f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, f32 ? 4 : 2, a.Cout, Mmax,
                 32, BM, f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B))
        return cudaErrorInvalidValue;
    }
    if (a.y32 && !(pair ? mat2d(&tmY32, a.y32, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.Cout, Mmax, 32, BM,
                                CU_TENSOR_MAP_SWIZZLE_64B)
                         : mat2d(&tmY32, a.y32, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, a.Cout, Mmax, 32, BM,
                                 CU_TENSOR_MAP_SWIZZLE_128B)))
      return cudaErrorInvalidValue;
    if (a.y && !mat2d(&tmY16, a.y, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.Cout, Mmax, 32, BM,
                      CU_TENSOR_MAP_SWIZZLE_64B))
      return cudaErrorInvalidValue;
  }
  const int smem = SMEM_MISC + pl.stages * CG<BN>::A_BYTES +
                   (pl.bres ? kblocks : pl.stages) * BB + (pl.staged ? 2 * EPI_WG : 0);
  if (cudaError_t e = ensure_smem(k_conv_gemm<BN, IM2COL, RT>, SMEM_LIMIT)) return e;
  const long long tiles = ((long long)Mmax + BM - 1) / BM * (a.Cout / BN);
  int grid = (int)(tiles < num_sms ? tiles : num_sms);
  if (grid < 1) grid = 1;
  k_conv_gemm<BN, IM2COL, RT><<<grid, THREADS, smem, stream>>>(tmA, tmB, tmR, tmY32, tmY16, tmA2, tmAL, tmRL, a, pl);
  return cudaGetLastError();
}

// row-tap form (k_conv_gemm RT): 3x3 / stride 1 / pad 1, whole samples per 128-row tile,
// image rows inside a warp, one 64-wide N tile (3 x 64 accumulator columns)
bool rowtap_ok(const ConvArgs& a) {
  const int hw = a.H * a.W;
  return a.ksz == 3 && a.stride == 1 && a.pad == 1 && a.Ho == a.H && a.Wo == a.W && hw <= BM && BM % hw == 0 &&
         32 % a.W == 0 && a.Cout == 64 && a.w_rt && a.Kp_rt == 3 * a.C && !a.x2 && !(a.dbg & (512 | 4194304));
}

template <int BN>
cudaError_t launch_bn(const ConvArgs& a, int max_rows, int num_sms, cudaStream_t stream) {
  if constexpr (BN == 64)
    if (rowtap_ok(a)) return launch_t<64, true, true>(a, max_rows, num_sms, stream);
  const bool tiled = a.ksz == 1 && a.stride == 1 && a.pad == 0;
  return tiled ? launch_t<BN, false>(a, max_rows, num_sms, stream) : launch_t<BN, true>(a, max_rows, num_sms, stream);
}

}  // namespace

bool conv_gemm_eligible(const ConvArgs& a) {
  const int k2 = a.x2 ? a.C2 : 0;
  if (a.x2 && (a.C2 % BKE || a.stride2 < 1 || a.stride2 > 8 || (a.H2 - 1) / a.stride2 + 1 != a.Ho ||
               (a.W2 - 1) / a.stride2 + 1 != a.Wo))
    return false;
  if (a.res_mode == 2 && (a.r_pad_lo % 4 || a.rC % 4 || a.rH < 2 * a.Ho || a.rW < 2 * a.Wo)) return false;
  if (a.rows_in || a.rows_out) {
    const int hw = a.Ho * a.Wo;
    if (hw > BM || BM % hw || hw % 8 || a.res_mode == 2 || a.x2) return false;
    if (a.rows_in && (a.ksz == 1 && a.stride == 1 && a.pad == 0)) return false;   // tiled A path: no list form
    if (a.rows_in && (a.H != a.Ho || a.W != a.Wo)) return false;
  }
  return a.nhwc && a.C % BKE == 0 && a.Cout % 64 == 0 && a.K == a.ksz * a.ksz * a.C + k2 && a.Kp == a.K &&
         a.pad <= 32 && a.stride <= 8 && (a.ksz > 1 || a.stride > 1 || a.H == a.Ho);
}

cudaError_t launch_conv_gemm(const ConvArgs& a, int max_rows, int num_sms, cudaStream_t stream) {
  if (!conv_gemm_eligible(a)) return cudaErrorNotSupported;
  // widest N tile that still gives every SM work when M is small (decode GEMMs: M = live rows)
  const long long m_tiles = ((long long)(max_rows > 0 ? max_rows : 1) * a.Ho * a.Wo + BM - 1) / BM;
  if (a.Cout % 256 == 0 && m_tiles * (a.Cout / 256) >= num_sms) return launch_bn<256>(a, max_rows, num_sms, stream);
  if (a.Cout % 128 == 0 && m_tiles * (a.Cout / 128) >= num_sms) return launch_bn<128>(a, max_rows, num_sms, stream);
  if (a.Cout % 256 == 0 && m_tiles * (a.Cout / 64) < num_sms / 2) return launch_bn<256>(a, max_rows, num_sms, stream);
  return launch_bn<64>(a, max_rows, num_sms, stream);
}

// Lazy-loading anchor: a kernel of this translation unit's module (preload_kernels, hostmod.cu).
__global__ void k_tu_anchor_conv_gemm() {}
const void* tu_anchor_conv_gemm() { return reinterpret_cast<const void*>(&k_tu_anchor_conv_gemm); }

}  // namespace dycl
