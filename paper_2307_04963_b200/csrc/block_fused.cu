// Fused residual basic block on tcgen05: y = relu(conv2(relu(conv1(x))) + x) for one
// whole sample at a time per CTA, stride 1, 3x3, C in {16, 32} (CIFAR stages 1-2).
//
// Why: per block the unfused kernels move x (bf16 operand copy), T (written + read),
// x (fp32 shortcut) and y (fp32 + bf16) through HBM: 256 KB per 32x32x16 sample.  Here
// the sample's fp32 residual stream is bulk-copied into SMEM once; the bf16 conv1
// operand is built from it in SMEM, T never leaves SMEM, the shortcut is read from SMEM,
// and only y (fp32, + a bf16 copy when the next layer needs one) is written: 128 KB.
//
// Operands use the row-tap form: per filter row r one tcgen05.mma with N = 3*C (the three
// W taps side by side), A = the sample's bf16 image in the UMMA K-major no-swizzle layout
// ([plane][H+2 rows][W][8 ch], two zero halo rows) shifted by r rows; the epilogue adds
// the three W-shifted partial sums with warp shuffles (pixel w-1 / w+1 = lane -1 / +1).
//
// SMEM banks: the epilogue owns one pixel per thread (TMEM lane = pixel), so plain NHWC
// fp32 rows (64 / 128 B apart) put 8 lanes of every LDS.128 phase in the same banks.  The
// fp32 sample is therefore moved by TMA with the 64B / 128B swizzle (16-byte chunk index
// XOR the 128-byte row index bits), read and written through swz(); y is written in place
// over its shortcut x and leaves through a tensor map that un-swizzles it.  The producer
// lane issues the stores and refills the buffer with the sample after next as soon as the
// stores have read it (double-buffered fp32 samples).
//
// Pipeline per sample i: convert(i+1) overlaps conv2(i); conv1(i+1) is issued sub-tile by
// sub-tile as epilogue 2(i) drains the shared TMEM accumulator (stage 1), or into its own
// accumulator set (stage 2).  Epilogue math uses packed f32x2 ops (combine16).
//
// Warps: 0-7 two epilogue/converter warpgroups (sub-tiles split even / odd), 8 bulk-copy
// producer, 9 TMEM allocator + MMA issuer.
#include <cuda.h>
#include <cuda_bf16.h>

#include "kernels.h"
#include "ptx.cuh"

namespace dycl {
namespace {

constexpr int THREADS = 352;          // 8 epilogue warps, sample producer, MMA, weight producer

template <int C, int H>
struct BCfg {
  static constexpr int W = H, HW = H * W, P = C / 8;
  static constexpr int NSUB = HW / 128;                 // UMMA tiles per sample
  static constexpr int BH = 128 / W;                    // image rows per UMMA tile
  static constexpr int N = 3 * C;                       // row-tap MMA width
  static constexpr int X32_BYTES = HW * C * 4;
  static constexpr int PLANE = (H + 2) * W * 16;        // one 8-channel plane with halo rows
  static constexpr int OPER = P * PLANE;                // bf16 operand image (x or T)
  static constexpr int KP_RT = (3 * C + 63) / 64 * 64;
  static constexpr int WCH = KP_RT / 8;                 // K chunks of the row-tap weights
  static constexpr int W_BYTES = WCH * N * 16;
  static constexpr int BOX_ROWS = HW < 256 ? HW : 256;  // pixels per TMA box (box dims <= 256)
  static constexpr int NBOX = HW / BOX_ROWS;
  // two weight slots (conv1 + conv2 of one block each), streamed block by block; biases of all
  // MAX_FUSED_BLOCKS blocks resident
  static constexpr int FIXED = 1024 + 2 * OPER + 2 * 2 * W_BYTES + 2 * MAX_FUSED_BLOCKS * C * 4 + 512 + 256 + 8 * C * 4;
  // fp32 sample buffers (2 if they fit: y is written in place over its own input x, which is
  // also the shortcut) and a separate bf16 output staging buffer if it fits
  static constexpr int NXB = FIXED + 2 * X32_BYTES <= 227 * 1024 ? 2 : 1;
  static constexpr int YB_BYTES = HW * C * 2;
  static constexpr bool YB_SEP = FIXED + NXB * X32_BYTES + YB_BYTES <= 227 * 1024;
  static constexpr int SMEM = FIXED + NXB * X32_BYTES + (YB_SEP ? YB_BYTES : 0);
  // separate TMEM accumulators for conv1 and conv2 if two fit: conv1(s+1) overlaps epilogue 2(s)
  static constexpr int NSETS = 2 * 256 >= 2 * NSUB * N && NSUB * N <= 256 ? 2 : 1;
  static_assert(HW % 128 == 0 && 128 % W == 0, "sample must tile into 128-row UMMA tiles");
  static_assert(NSUB * N <= 512, "TMEM");
  static_assert(SMEM <= 227 * 1024, "SMEM");
  static_assert(NXB == 2, "y is staged in place over x: the next sample needs the other buffer");
};

// byte offset inside a swizzled fp32 sample buffer (1024-aligned): C=32 -> 128B swizzle,
// C=16 -> 64B swizzle (CU_TENSOR_MAP_SWIZZLE_128B / _64B patterns)
template <int C>
__device__ __forceinline__ uint32_t swz(uint32_t o) {
  return C == 32 ? o ^ (((o >> 7) & 7u) << 4) : o ^ (((o >> 7) & 3u) << 4);
}

__device__ __forceinline__ uint32_t pk(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Refill a sample buffer box by box: box q is reloaded once the bulk store group of box q
// (committed in order, one group per box) has read it (cp.async.bulk.wait_group.read NBOX-1-q).
template <int NB, int Q = 0, typename F>
__device__ __forceinline__ void refill(F&& load_box) {
  if constexpr (Q < NB) {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NB - 1 - Q) : "memory");
    load_box(Q);
    refill<NB, Q + 1>(load_box);
  }
}

// Row-tap combine of 16 channels of one pixel (TMEM lane = pixel w of an image row, lanes of a
// warp = consecutive pixels): f = relu(D1(w) + bias [+ res] + D0(w-1) + D2(w+1)), the W
// neighbours by warp shuffle, masked at the row ends by a 0/1 FMA factor; res(q) returns the
// shortcut channels q..q+3 (read from SMEM just in time).  Packed f32x2 ops
// (FADD2 / FFMA2) halve the instruction count; every term is added with one fp32 rounding.
template <int W, typename Res>
__device__ __forceinline__ void combine16(const uint32_t (&v)[3][16], int w, const float* bias, Res res,
                                          float (&f)[16], bool with_res = true) {
  const float ml = w > 0 ? 1.0f : 0.0f, mr = w < W - 1 ? 1.0f : 0.0f;
  const float2 ml2 = make_float2(ml, ml), mr2 = make_float2(mr, mr);
#pragma unroll
  for (int q = 0; q < 16; q += 4) {
    const float4 b4 = *reinterpret_cast<const float4*>(bias + q);
    float2 t0 = __fadd2_rn(make_float2(__uint_as_float(v[1][q]), __uint_as_float(v[1][q + 1])), make_float2(b4.x, b4.y));
    float2 t1 = __fadd2_rn(make_float2(__uint_as_float(v[1][q + 2]), __uint_as_float(v[1][q + 3])), make_float2(b4.z, b4.w));
    if (with_res) {
      const float4 r4 = res(q);
      t0 = __fadd2_rn(t0, make_float2(r4.x, r4.y));
      t1 = __fadd2_rn(t1, make_float2(r4.z, r4.w));
    }
    float l[4], rr[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      l[k] = __shfl_up_sync(0xffffffffu, __uint_as_float(v[0][q + k]), 1);
      rr[k] = __shfl_down_sync(0xffffffffu, __uint_as_float(v[2][q + k]), 1);
    }
    t0 = __ffma2_rn(make_float2(l[0], l[1]), ml2, t0);
    t1 = __ffma2_rn(make_float2(l[2], l[3]), ml2, t1);
    t0 = __ffma2_rn(make_float2(rr[0], rr[1]), mr2, t0);
    t1 = __ffma2_rn(make_float2(rr[2], rr[3]), mr2, t1);
    f[q] = fmaxf(t0.x, 0.f);
    f[q + 1] = fmaxf(t0.y, 0.f);
    f[q + 2] = fmaxf(t1.x, 0.f);
    f[q + 3] = fmaxf(t1.y, 0.f);
  }
}

struct WMaps {
  CUtensorMap m[2 * MAX_FUSED_BLOCKS];   // conv1, conv2 row-tap weights of each fused block
};

template <int C, int H>
__global__ void __launch_bounds__(THREADS, 1)
    k_block_fused(const __grid_constant__ WMaps wm, const __grid_constant__ CUtensorMap tmX,
                  const __grid_constant__ CUtensorMap tmY, const BlockArgs a) {
  using G = BCfg<C, H>;
  constexpr int W = G::W, HW = G::HW, P = G::P;
  const int NB = a.nblk;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* x32s = smem;                                                   // [NXB][HW][C] fp32, swizzled (x, then y)
  uint8_t* xb = x32s + G::NXB * G::X32_BYTES;                             // [P][H+2][W][8] bf16
  uint8_t* tb = xb + G::OPER;
  uint8_t* ws = tb + G::OPER;                                             // [2 slots][conv1, conv2] row-tap weights
  uint8_t* ybs = ws + 2 * 2 * G::W_BYTES;                                 // [P][HW][8] bf16 y staging
  float* bs = reinterpret_cast<float*>(ybs + (G::YB_SEP ? G::YB_BYTES : 0));   // [MAX_FUSED_BLOCKS][b1 | b2]
  uint64_t* bars = reinterpret_cast<uint64_t*>(bs + 2 * MAX_FUSED_BLOCKS * C);
  // yready[b][k]: box k of buffer b holds y (both warpgroups arrived)
  const uint32_t xfull0 = ptx::smem_u32(bars), yready0 = ptx::smem_u32(bars + 26);
  const uint32_t xb_full = xfull0 + 16, xb_empty = xb_full + 8, acc1 = xb_empty + 8, tb_full = acc1 + 8;
  const uint32_t acc2 = tb_full + 8, acc1_empty = acc2 + 8, wfull = acc1_empty + 8, acc2_empty = wfull + 8;
  const uint32_t tb_free = acc2_empty + 8;             // the bf16-copy store has read T / ybs
  const uint32_t subfree0 = acc2_empty + 16;          // [NSUB] shared set: sub-tile j drained by epilogue 2
  // per sub-tile j: conv1 / conv2 accumulator j complete (MMA commit), and tready[j] = epilogue 1
  // has read accumulator j and written T rows of sub-tile j (conv2 sub-tile j needs j-1..j+1)
  const uint32_t acc1j0 = ptx::smem_u32(bars + 34), acc2j0 = ptx::smem_u32(bars + 42), tready0 = ptx::smem_u32(bars + 50);
  // weight ring: wfull[s] = slot s loaded (TMA), wempty[s] = conv2 of the block in slot s done
  const uint32_t wfull0 = ptx::smem_u32(bars + 58), wempty0 = ptx::smem_u32(bars + 60);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 62);
  // xready[j]: between fused blocks, epilogue 2 wrote the bf16 operand rows of sub-tile j (the
  // next conv1 sub-tile j needs j-1..j+1): the next block starts before this one's epilogue ends
  const uint32_t xready0 = ptx::smem_u32(bars + 66);
  float* gred = reinterpret_cast<float*>(bars + 74);       // [8 warps][C] fused-GAP partials (C <= 32)
  static_assert(G::NBOX <= 4, "box barriers");
  static_assert(G::NSUB <= 8, "sub-tile barriers");
  constexpr uint32_t SET2 = G::NSETS == 2 ? 256u : 0u;    // TMEM column of the conv2 accumulator

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_live = a.n_live ? *a.n_live : a.n_static;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(xfull0 + 8 * i, 1);
      for (int k = 0; k < G::NBOX; ++k) ptx::mbar_init(yready0 + 8 * (4 * i + k), 256);
    }
    ptx::mbar_init(tb_free, 1);
    for (int j = 0; j < G::NSUB; ++j) {
      ptx::mbar_init(subfree0 + 8 * j, 128);
      ptx::mbar_init(acc1j0 + 8 * j, 1);
      ptx::mbar_init(acc2j0 + 8 * j, 1);
      ptx::mbar_init(tready0 + 8 * j, 128);
      ptx::mbar_init(xready0 + 8 * j, 128);
    }
    ptx::mbar_init(xb_full, 256);
    ptx::mbar_init(xb_empty, 1);
    ptx::mbar_init(acc1, 1);
    ptx::mbar_init(tb_full, 256);
    ptx::mbar_init(acc2, 1);
    ptx::mbar_init(acc1_empty, 256);
    ptx::mbar_init(acc2_empty, 256);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(wfull0 + 8 * i, 1);
      ptx::mbar_init(wempty0 + 8 * i, 1);
    }
    ptx::fence_mbar_init();
  }
  // zero the halo rows (row 0 and row H+1 of every plane) of both operand images, once
  for (int i = threadIdx.x; i < 2 * P * 2 * W; i += blockDim.x) {
    const int img = i / (P * 2 * W), rem = i % (P * 2 * W);
    const int p = rem / (2 * W), k = rem % (2 * W);
    const int row = k < W ? 0 : H + 1, w = k % W;
    uint8_t* base = img ? tb : xb;
    *reinterpret_cast<uint4*>(base + p * G::PLANE + (row * W + w) * 16) = make_uint4(0, 0, 0, 0);
  }
  for (int i = threadIdx.x; i < 2 * NB * C; i += blockDim.x) {
    const int blk = i / (2 * C), k = (i / C) & 1, c = i % C;
    bs[i] = (k ? a.b2[blk] : a.b1[blk])[c];
  }
  ptx::fence_proxy_async_smem();
  if (warp == 9) ptx::tmem_alloc(ptx::smem_u32(tmem_slot), 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tmX);
      // The producer owns both fp32 sample buffers: it loads sample it into buffer it % 2, and
      // once the epilogue has written y over it (yready), stores y (+ the bf16 copy), waits for
      // the stores to have READ SMEM and refills the buffer with sample it + 2 right away.
      auto load = [&](int k) {
        const int smp = blockIdx.x + k * gridDim.x;
        if (smp >= n_live) return;
        const int b = k % G::NXB;
        if (a.ts && blockIdx.x == 0 && k < 8) a.ts[k * 16 + 10] = clock64();
        const int src = a.list ? a.list[smp] : smp;
        ptx::mbar_arrive_expect_tx(xfull0 + 8 * b, G::X32_BYTES);
#pragma unroll
        for (int q = 0; q < G::NBOX; ++q)
          ptx::tma_load_2d(ptx::smem_u32(x32s + (size_t)b * G::X32_BYTES + q * G::BOX_ROWS * C * 4), &tmX,
                           xfull0 + 8 * b, 0, src * HW + q * G::BOX_ROWS);
      };
      load(0);
      load(1);
      int it = 0;
      for (int smp = blockIdx.x; smp < n_live; smp += gridDim.x, ++it) {
        const int b = it % G::NXB;
        const uint8_t* xs = x32s + (size_t)b * G::X32_BYTES;
        const int dst = a.list && a.list_out ? a.list[smp] : smp;   // dense order, or in place
        // store box by box as epilogue 2 finishes it (one bulk group per box) ...
#pragma unroll
        for (int q = 0; q < G::NBOX; ++q) {
          ptx::mbar_wait(yready0 + 8 * (4 * b + q), (it / G::NXB) & 1);
          if (a.yb)
            for (int p = 0; p < P; ++p)
              ptx::bulk_store(a.yb + (size_t)dst * C * HW + (size_t)p * HW * 8 + (size_t)q * G::BOX_ROWS * 8,
                              ptx::smem_u32((G::YB_SEP ? ybs + p * HW * 16 : tb + p * G::PLANE + W * 16) +
                                            q * G::BOX_ROWS * 16),
                              G::BOX_ROWS * 16);
          ptx::tma_store_2d(&tmY, ptx::smem_u32(xs + q * G::BOX_ROWS * C * 4), 0, dst * HW + q * G::BOX_ROWS);
          ptx::bulk_commit();
        }
        // ... and refill the buffer box by box with sample it + 2 as the stores read it out
        const int nsmp = blockIdx.x + (it + 2) * gridDim.x;
        if (nsmp < n_live) {
          if (a.ts && blockIdx.x == 0 && it + 2 < 8) a.ts[(it + 2) * 16 + 10] = clock64();
          const int src = a.list ? a.list[nsmp] : nsmp;
          ptx::mbar_arrive_expect_tx(xfull0 + 8 * b, G::X32_BYTES);
          refill<G::NBOX>([&](int q) {
            ptx::tma_load_2d(ptx::smem_u32(x32s + (size_t)b * G::X32_BYTES + q * G::BOX_ROWS * C * 4), &tmX,
                             xfull0 + 8 * b, 0, src * HW + q * G::BOX_ROWS);
          });
        } else {
          ptx::bulk_wait_read0();
        }
        ptx::mbar_arrive(tb_free);                   // all stores have read T / ybs
      }
      ptx::bulk_wait0();                             // y writes complete before the CTA retires
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer
    // conv occurrence k = it * NB + blk: conv1 / conv2 of fused block blk of this CTA's
    // it-th sample; every barrier below completes once per occurrence.
    constexpr uint32_t IDESC = ptx::make_idesc_bf16(128, G::N);
    const uint64_t xdesc = ptx::make_smem_desc(ptx::smem_u32(xb), 0, G::PLANE, 128);
    const uint64_t tdesc = ptx::make_smem_desc(ptx::smem_u32(tb), 0, G::PLANE, 128);
    int it = 0;
    for (int smp = blockIdx.x; smp < n_live; smp += gridDim.x, ++it) {
      const bool mstamp = a.ts && blockIdx.x == 0 && lane == 0 && it < 8;
      for (int blk = 0; blk < NB; ++blk) {
        const int k = it * NB + blk;
        const uint32_t ph = k & 1;
        // weight slot of this occurrence: resident per block when NB <= 2, else the ring
        const bool wres = NB <= 2;
        const int ws_slot = wres ? blk : (k & 1);
        ptx::mbar_wait(wfull0 + 8 * ws_slot, wres ? 0u : (uint32_t)((k >> 1) & 1));
        const uint64_t w1d = ptx::make_smem_desc(ptx::smem_u32(ws + (2 * ws_slot) * G::W_BYTES), 0, G::N * 16, 128);
        const uint64_t w2d =
            ptx::make_smem_desc(ptx::smem_u32(ws + (2 * ws_slot + 1) * G::W_BYTES), 0, G::N * 16, 128);
        // conv1 sub-tile j: its columns were drained by the previous epilogue 2 (shared set) or the
        // previous epilogue 1 (two sets); committed per sub-tile so epilogue 1 starts on sub-tile 0
        // while the tensor core works on the rest
        // x operand: the converted sample (first block) or, sub-tile by sub-tile below, the
        // previous block's y
        const uint32_t pxr = (uint32_t)((it * (NB - 1) + blk - 1) & 1);
        if (blk == 0) ptx::mbar_wait(xb_full, it & 1);
        ptx::tc_fence_after();
        if (mstamp && blk == 0) a.ts[it * 16 + 6] = clock64();
#pragma unroll
        for (int j = 0; j < G::NSUB; ++j) {
          if (blk > 0) {
            if (j == 0) ptx::mbar_wait(xready0, pxr);
            if (j + 1 < G::NSUB) ptx::mbar_wait(xready0 + 8 * (j + 1), pxr);
          }
          if (k > 0) ptx::mbar_wait((G::NSETS == 1 ? subfree0 : tready0) + 8 * j, (k - 1) & 1);
          if (k > 0 || blk > 0) ptx::tc_fence_after();
          // one elected lane issues the sub-tile's MMAs; descriptors advance by 32-bit adds on
          // their start-address word (a per-MMA elect + 64-bit descriptor build cost more issue
          // slots than a 128 x 3C x 16 MMA runs)
          if (ptx::elect_one()) {
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
              for (int q = 0; q < C / 16; ++q)
                ptx::mma_bf16_ss_lohi(tmem + j * G::N,
                                      (uint32_t)xdesc + (uint32_t)(((j * G::BH + r) * W * 16 + 2 * q * G::PLANE) >> 4),
                                      (uint32_t)(xdesc >> 32),
                                      (uint32_t)w1d + (uint32_t)(((r * P + 2 * q) * G::N * 16) >> 4),
                                      (uint32_t)(w1d >> 32), IDESC, (uint32_t)((r | q) != 0));
          }
          __syncwarp();
          ptx::mma_commit_elect(acc1j0 + 8 * j);
        }
        // xb is free for the next sample's conversion once the LAST block's conv1 has read it
        // (earlier blocks' reads are ordered before the epilogue-2 writes that refill xb by the
        // acc2 commit, which covers every prior MMA): one completion per sample, no skipped phase
        if (blk == NB - 1) ptx::mma_commit_elect(xb_empty);
        __syncwarp();
        if (mstamp && blk == 0) a.ts[it * 16 + 7] = clock64();
        if (mstamp && blk == NB - 1) a.ts[it * 16 + 8] = clock64();
        // conv2 sub-tile j: T rows of sub-tiles j-1..j+1 written (and, shared set, accumulator j
        // read) by epilogue 1; two sets: SET2 columns j drained by the previous epilogue 2
#pragma unroll
        for (int j = 0; j < G::NSUB; ++j) {
          // T rows j-1..j+1: j-1 and j were already awaited for sub-tile j-1 (each barrier
          // completes once per occurrence), so only the new neighbour j+1 is waited on
          if (j == 0) ptx::mbar_wait(tready0, ph);
          if (j + 1 < G::NSUB) ptx::mbar_wait(tready0 + 8 * (j + 1), ph);
          if (G::NSETS == 2 && k > 0) ptx::mbar_wait(subfree0 + 8 * j, (k - 1) & 1);
          ptx::tc_fence_after();
          if (ptx::elect_one()) {
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
              for (int q = 0; q < C / 16; ++q)
                ptx::mma_bf16_ss_lohi(tmem + SET2 + j * G::N,
                                      (uint32_t)tdesc + (uint32_t)(((j * G::BH + r) * W * 16 + 2 * q * G::PLANE) >> 4),
                                      (uint32_t)(tdesc >> 32),
                                      (uint32_t)w2d + (uint32_t)(((r * P + 2 * q) * G::N * 16) >> 4),
                                      (uint32_t)(w2d >> 32), IDESC, (uint32_t)((r | q) != 0));
          }
          __syncwarp();
          ptx::mma_commit_elect(acc2j0 + 8 * j);
        }
        if (!wres) ptx::mma_commit_elect(wempty0 + 8 * ws_slot);   // free the ring slot once conv2 ends
        __syncwarp();
        if (mstamp && blk == NB - 1) a.ts[it * 16 + 9] = clock64();
      }
    }
  } else if (warp == 10) {
    // ------------------------------------------------------------ weight producer
    // the fused blocks' weights stream through two SMEM slots, one block ahead of the MMA
    if (lane == 0 && NB <= 2) {                      // resident: each block's weights once
      for (int blk = 0; blk < NB; ++blk) {
        ptx::mbar_arrive_expect_tx(wfull0 + 8 * blk, 2 * G::W_BYTES);
#pragma unroll
        for (int h = 0; h < 2; ++h)
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
              "%5}], [%2];" ::"r"(ptx::smem_u32(ws + (2 * blk + h) * G::W_BYTES)),
              "l"(&wm.m[2 * blk + h]), "r"(wfull0 + 8 * blk), "r"(0), "r"(0), "r"(0)
              : "memory");
      }
    } else if (lane == 0) {
      int k = 0;
      for (int smp = blockIdx.x; smp < n_live; smp += gridDim.x)
        for (int blk = 0; blk < NB; ++blk, ++k) {
          const int sl = k & 1;
          if (k >= 2) ptx::mbar_wait(wempty0 + 8 * sl, ((k - 2) >> 1) & 1);
          ptx::mbar_arrive_expect_tx(wfull0 + 8 * sl, 2 * G::W_BYTES);
#pragma unroll
          for (int h = 0; h < 2; ++h)
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
                "%5}], [%2];" ::"r"(ptx::smem_u32(ws + (2 * sl + h) * G::W_BYTES)),
                "l"(&wm.m[2 * blk + h]), "r"(wfull0 + 8 * sl), "r"(0), "r"(0), "r"(0)
                : "memory");
        }
    }
  } else {
    // ------------------------------------------------------------ converters / epilogues
    const int wg = warp >> 2, quad = warp & 3;
    const int r = quad * 32 + lane;                    // TMEM lane = row of a UMMA tile
    const int et = threadIdx.x;                        // 0..255
    const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
    constexpr int CPS = C / 16;                        // 16-channel chunks per sub-tile
    constexpr int UPT = (G::NSUB / 2) * CPS;           // (sub-tile, chunk) units per thread
    static_assert(UPT % 2 == 0, "units are processed in pairs");

    // fp32 stream -> bf16 operand image (RNE); frees the fp32 input buffer
    auto convert = [&](int itc) {
      const int b = itc % G::NXB;
      const uint8_t* xs = x32s + (size_t)b * G::X32_BYTES;
      ptx::mbar_wait(xfull0 + 8 * b, (itc / G::NXB) & 1);
      ptx::mbar_wait(xb_empty, (itc - 1) & 1);         // the previous sample's last conv1 read xb
#pragma unroll 4
      for (int u = et; u < HW * P; u += 256) {
        const int pix = u % HW, p = u / HW;            // lanes = consecutive pixels (swizzled rows)
        const float4 v0 = *reinterpret_cast<const float4*>(xs + swz<C>((uint32_t)(pix * C + p * 8) * 4));
        const float4 v1 = *reinterpret_cast<const float4*>(xs + swz<C>((uint32_t)(pix * C + p * 8 + 4) * 4));
        *reinterpret_cast<uint4*>(xb + p * G::PLANE + (W + pix) * 16) =
            make_uint4(pk(v0.x, v0.y), pk(v0.z, v0.w), pk(v1.x, v1.y), pk(v1.z, v1.w));
      }
      ptx::fence_proxy_async_smem();
      ptx::mbar_arrive(xb_full);              // x32s[b] stays: it is the shortcut and y's staging
    };

    int it = 0;
    if ((int)blockIdx.x < n_live) convert(0);
    for (int smp = blockIdx.x; smp < n_live; smp += gridDim.x, ++it) {
     for (int blk = 0; blk < NB; ++blk) {
      const int kocc = it * NB + blk;
      const uint32_t ph = kocc & 1;
      const bool last = blk == NB - 1;
      const float* b1s = bs + 2 * blk * C;
      const float* b2s = b1s + C;
      const bool stamp = a.ts && blockIdx.x == 0 && et == 0 && it < 8;
      // ---- epilogue 1: T = relu(conv1 + b1) -> bf16 operand image (SMEM), sub-tile by sub-tile
      // as the conv1 accumulators complete
      // the previous sample's bf16-copy store (from T / ybs) has read SMEM: T / ybs may be rewritten
      if (blk == 0 && it > 0 && a.yb) ptx::mbar_wait(tb_free, (it - 1) & 1);
      if (stamp && blk == 0) a.ts[it * 16 + 2] = clock64();
#pragma unroll
      for (int g = 0; g < UPT; g += 2) {
        uint32_t v[2][3][16];
        const int ja = wg + 2 * (g / CPS), jb = wg + 2 * ((g + 1) / CPS);   // sub-tiles of this pair
        ptx::mbar_wait(acc1j0 + 8 * ja, ph);
        if (jb != ja) ptx::mbar_wait(acc1j0 + 8 * jb, ph);
        ptx::tc_fence_after();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int j = wg + 2 * ((g + u) / CPS), c0 = ((g + u) % CPS) * 16;
          const uint32_t t = lane_base + (uint32_t)(j * G::N + c0);
          ptx::tmem_ld_32x32b_x16(t, v[u][0]);
          ptx::tmem_ld_32x32b_x16(t + C, v[u][1]);
          ptx::tmem_ld_32x32b_x16(t + 2 * C, v[u][2]);
        }
        ptx::tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int j = wg + 2 * ((g + u) / CPS), c0 = ((g + u) % CPS) * 16;
          const int pix = j * 128 + r, w = pix % W;
          float f[16];
          combine16<W>(v[u], w, b1s + c0, [](int) { return make_float4(0.f, 0.f, 0.f, 0.f); }, f, false);
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2)
            *reinterpret_cast<uint4*>(tb + ((c0 >> 3) + h2) * G::PLANE + (W + pix) * 16) =
                make_uint4(pk(f[8 * h2], f[8 * h2 + 1]), pk(f[8 * h2 + 2], f[8 * h2 + 3]),
                           pk(f[8 * h2 + 4], f[8 * h2 + 5]), pk(f[8 * h2 + 6], f[8 * h2 + 7]));
        }
        // T rows of these sub-tiles written, their accumulators read: conv2 may use / reuse them
        ptx::fence_proxy_async_smem();
        ptx::tc_fence_before();
        ptx::mbar_arrive(tready0 + 8 * ja);
        if (jb != ja) ptx::mbar_arrive(tready0 + 8 * jb);
      }
      if (stamp && blk == 0) a.ts[it * 16 + 3] = clock64();
      // ---- next sample's operand conversion overlaps the last conv2 of this one
      if (last && smp + (int)gridDim.x < n_live) {
        if (stamp) a.ts[(it + 1) * 16 + 0] = clock64();
        convert(it + 1);
        if (stamp) a.ts[(it + 1) * 16 + 1] = clock64();
      }
      // ---- epilogue 2: y = relu(conv2 + b2 + x) -> fp32 stream (+ bf16 operand copy); the
      // shortcut x is this sample's fp32 buffer in SMEM and y overwrites it in place
      uint8_t* xs = x32s + (size_t)(it % G::NXB) * G::X32_BYTES;
      if (stamp && last) a.ts[it * 16 + 4] = clock64();
#pragma unroll
      for (int g = 0; g < UPT; g += 2) {
        uint32_t v[2][3][16];
        const int ja = wg + 2 * (g / CPS), jb = wg + 2 * ((g + 1) / CPS);
        ptx::mbar_wait(acc2j0 + 8 * ja, ph);
        if (jb != ja) ptx::mbar_wait(acc2j0 + 8 * jb, ph);
        ptx::tc_fence_after();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int j = wg + 2 * ((g + u) / CPS), c0 = ((g + u) % CPS) * 16;
          const uint32_t t = lane_base + SET2 + (uint32_t)(j * G::N + c0);
          ptx::tmem_ld_32x32b_x16(t, v[u][0]);
          ptx::tmem_ld_32x32b_x16(t + C, v[u][1]);
          ptx::tmem_ld_32x32b_x16(t + 2 * C, v[u][2]);
        }
        ptx::tmem_ld_wait();
        // these sub-tiles' conv2 columns are read: the next conv1 (shared set) / conv2 (two sets) may reuse them
        ptx::tc_fence_before();
        ptx::mbar_arrive(subfree0 + 8 * ja);
        if (jb != ja) ptx::mbar_arrive(subfree0 + 8 * jb);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int j = wg + 2 * ((g + u) / CPS), c0 = ((g + u) % CPS) * 16;
          const int pix = j * 128 + r, w = pix % W;
          float f[16];
          combine16<W>(v[u], w, b2s + c0, [&](int q) {
            return *reinterpret_cast<const float4*>(xs + swz<C>((uint32_t)(pix * C + c0 + q) * 4));
          }, f);
          // y overwrites its own shortcut x in place (the producer TMA-stores it)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *reinterpret_cast<float4*>(xs + swz<C>((uint32_t)(pix * C + c0 + 4 * q) * 4)) =
                make_float4(f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
          if (!last) {                                 // the next fused block's conv1 operand
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2)
              *reinterpret_cast<uint4*>(xb + ((c0 >> 3) + h2) * G::PLANE + (W + pix) * 16) =
                  make_uint4(pk(f[8 * h2], f[8 * h2 + 1]), pk(f[8 * h2 + 2], f[8 * h2 + 3]),
                             pk(f[8 * h2 + 4], f[8 * h2 + 5]), pk(f[8 * h2 + 6], f[8 * h2 + 7]));
          } else if (a.yb) {
            uint8_t* yb_pl = G::YB_SEP ? ybs : tb + W * 16;     // plane stride: HW*16 / PLANE
            constexpr int PSTR = G::YB_SEP ? HW * 16 : G::PLANE;
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2)
              *reinterpret_cast<uint4*>(yb_pl + ((c0 >> 3) + h2) * PSTR + pix * 16) =
                  make_uint4(pk(f[8 * h2], f[8 * h2 + 1]), pk(f[8 * h2 + 2], f[8 * h2 + 3]),
                             pk(f[8 * h2 + 4], f[8 * h2 + 5]), pk(f[8 * h2 + 6], f[8 * h2 + 7]));
          }
          if (last && !a.pooled && c0 + 16 == C) {     // sub-tile j done: hand its box to the producer
            ptx::fence_proxy_async_smem();
            ptx::mbar_arrive(yready0 + 8 * (4 * (it % G::NXB) + j * 128 / G::BOX_ROWS));
          }
        }
        if (!last) {                                   // y (bf16) rows: the next block's conv1 operand
          ptx::fence_proxy_async_smem();
          ptx::mbar_arrive(xready0 + 8 * ja);
          if (jb != ja) ptx::mbar_arrive(xready0 + 8 * jb);
        }
      }
      if (last && a.pooled) {
        // global average pool of y for the head that follows (a2 fused): y sits in SMEM; thread t
        // sums channel quad t % (C/4) over pixels t / (C/4), + 256/(C/4), ...; lanes sharing a
        // quad reduce by shuffles, warps through SMEM, fixed order throughout
        constexpr int NQ = C / 4, PST = 256 / NQ;
        asm volatile("bar.sync 1, 256;" ::: "memory");
        const int cq = et % NQ;
        float4 acc4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
        for (int pix = et / NQ; pix < HW; pix += PST) {
          const float4 q = *reinterpret_cast<const float4*>(xs + swz<C>((uint32_t)(pix * C + 4 * cq) * 4));
          acc4.x += q.x; acc4.y += q.y; acc4.z += q.z; acc4.w += q.w;
        }
#pragma unroll
        for (int o = NQ; o < 32; o <<= 1) {
          acc4.x += __shfl_xor_sync(0xffffffffu, acc4.x, o);
          acc4.y += __shfl_xor_sync(0xffffffffu, acc4.y, o);
          acc4.z += __shfl_xor_sync(0xffffffffu, acc4.z, o);
          acc4.w += __shfl_xor_sync(0xffffffffu, acc4.w, o);
        }
        if (lane < NQ) *reinterpret_cast<float4*>(gred + (warp * NQ + lane) * 4) = acc4;
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (et < C) {
          float sum = 0.f;
#pragma unroll
          for (int w8 = 0; w8 < 8; ++w8) sum += gred[(w8 * NQ + et / 4) * 4 + (et & 3)];
          const int dst = a.list && a.list_out ? a.list[smp] : smp;
          a.pooled[(size_t)dst * C + et] = sum * (1.0f / HW);
        }
        ptx::fence_proxy_async_smem();
#pragma unroll
        for (int q = 0; q < G::NBOX; ++q) ptx::mbar_arrive(yready0 + 8 * (4 * (it % G::NXB) + q));
      }
      if (stamp && last) a.ts[it * 16 + 5] = clock64();
     }
    }

  }
  __syncthreads();
  if (warp == 9) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn enc_fn() {
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

template <int C, int H>
cudaError_t launch_ch(const BlockArgs& a, int max_rows, int num_sms, cudaStream_t stream) {
  using G = BCfg<C, H>;
  EncodeTiledFn enc = enc_fn();
  if (!enc) return cudaErrorNotSupported;
  WMaps wm;
  for (int i = 0; i < 2 * a.nblk; ++i) {
    const uint16_t* w = (i & 1) ? a.w2_rt[i / 2] : a.w1_rt[i / 2];
    cuuint64_t dims[3] = {8, (cuuint64_t)G::N, (cuuint64_t)G::WCH};
    cuuint64_t strides[2] = {(cuuint64_t)G::KP_RT * 2, 16};
    cuuint32_t box[3] = {8, (cuuint32_t)G::N, (cuuint32_t)G::WCH};
    cuuint32_t es[3] = {1, 1, 1};
    if (enc(&wm.m[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, (void*)w, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  // fp32 stream in / out: [rows][C] fp32, box [BOX_ROWS][C], swizzled to the C*4-byte row
  CUtensorMap tm[2];
  const float* xy[2] = {a.x32, a.y32};
  for (int i = 0; i < 2; ++i) {
    cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)max_rows * G::HW};
    cuuint64_t strides[1] = {(cuuint64_t)C * 4};
    cuuint32_t box[2] = {(cuuint32_t)C, (cuuint32_t)G::BOX_ROWS};
    cuuint32_t es[2] = {1, 1};
    if (enc(&tm[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)xy[i], dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, C == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  if (cudaError_t e = ensure_smem(k_block_fused<C, H>, G::SMEM)) return e;
  int grid = max_rows < num_sms ? max_rows : num_sms;
  if (grid < 1) grid = 1;
  k_block_fused<C, H><<<grid, THREADS, G::SMEM, stream>>>(wm, tm[0], tm[1], a);
  return cudaGetLastError();
}

}  // namespace

bool block_fused_eligible(int C, int H, int W) { return H == W && ((C == 16 && H == 32) || (C == 32 && H == 16)); }

cudaError_t launch_block_fused(const BlockArgs& a, int max_rows, int num_sms, cudaStream_t stream) {
  if (a.nblk < 1 || a.nblk > MAX_FUSED_BLOCKS) return cudaErrorInvalidValue;
  if (a.C == 16 && a.H == 32 && a.W == 32) return launch_ch<16, 32>(a, max_rows, num_sms, stream);
  if (a.C == 32 && a.H == 16 && a.W == 16) return launch_ch<32, 16>(a, max_rows, num_sms, stream);
  return cudaErrorNotSupported;
}

// Lazy-loading anchor: a kernel of this translation unit's module (preload_kernels, hostmod.cu).
__global__ void k_tu_anchor_block_fused() {}
const void* tu_anchor_block_fused() { return reinterpret_cast<const void*>(&k_tu_anchor_block_fused); }

}  // namespace dycl
