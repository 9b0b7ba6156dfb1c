// Device-side host module: pre-processing cast, heads + per-sample predicates,
// stable compaction, scatter to original order, row gathers.
//
// The paper's host program evaluates each `If` node on the host after copying the
// predicate tensor back (Listing 2 set_input/run/get_output, PAPER.md L216-218;
// the transfer overhead is Challenge 2, L499-501).  Here every logic node runs
// on the device and writes its decisions as index lists + device-resident counts
// that the next kernels read, so a whole batched run needs no host round trip.
// All reductions use fixed-order trees (no atomics), so results are independent
// of batch size and of the position of a sample in the batch.
#include <cuda.h>
#include <cuda_bf16.h>

#include <map>
#include <mutex>
#include <set>
#include <vector>

#include "epilogue.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace dycl {

cudaError_t ensure_smem(const void* func, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = done[{dev, func}];
  if (cur >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}

cudaError_t preload_kernels() {
  typedef CUresult (*FuncGetModule)(CUmodule*, CUfunction);
  typedef CUresult (*ModuleGetFunctionCount)(unsigned int*, CUmodule);
  typedef CUresult (*ModuleEnumerateFunctions)(CUfunction*, unsigned int, CUmodule);
  typedef CUresult (*FuncLoad)(CUfunction);
  static std::mutex mu;
  static std::set<int> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(dev)) return cudaSuccess;
  auto sym = [](const char* name) -> void* {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    return cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess &&
                   q == cudaDriverEntryPointSuccess
               ? p
               : nullptr;
  };
  auto get_module = reinterpret_cast<FuncGetModule>(sym("cuFuncGetModule"));
  auto count = reinterpret_cast<ModuleGetFunctionCount>(sym("cuModuleGetFunctionCount"));
  auto enumerate = reinterpret_cast<ModuleEnumerateFunctions>(sym("cuModuleEnumerateFunctions"));
  auto load = reinterpret_cast<FuncLoad>(sym("cuFuncLoad"));
  if (!get_module || !count || !enumerate || !load) return cudaErrorNotSupported;
  const void* anchors[] = {tu_anchor_conv_tc(), tu_anchor_conv_tma(),   tu_anchor_conv_gemm(), tu_anchor_conv_halo(),
                           tu_anchor_gemm_tma(), tu_anchor_block_fused(), tu_anchor_hostmod(),  tu_anchor_s2s_kernels(),
                           tu_anchor_cap(),      tu_anchor_drb()};
  for (const void* a : anchors) {
    cudaFunction_t f = nullptr;
    if ((e = cudaGetFuncBySymbol(&f, a)) != cudaSuccess) return e;
    CUmodule m = nullptr;
    unsigned n = 0;
    if (get_module(&m, reinterpret_cast<CUfunction>(f)) != CUDA_SUCCESS || count(&n, m) != CUDA_SUCCESS)
      return cudaErrorNotSupported;
    std::vector<CUfunction> fs(n);
    if (n && enumerate(fs.data(), n, m) != CUDA_SUCCESS) return cudaErrorNotSupported;
    for (CUfunction fn : fs)
      if (load(fn) != CUDA_SUCCESS) return cudaErrorNotSupported;
  }
  done.insert(dev);
  return cudaSuccess;
}

namespace {

__device__ __forceinline__ float bf16f(uint16_t u) { return __uint_as_float((uint32_t)u << 16); }

// ------------------------------------------------------------------ a0 cast
// fp32 NHWC [n][hw][c] -> bf16 channel-planar [n][cp/8][hw][8] (channels >= c zero).
__global__ void k_cast_pad(const float* __restrict__ in, uint16_t* __restrict__ out, int64_t npix, int hw, int c,
                           int cp) {
  const int planes = cp / 8;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < npix * planes;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gp = u % npix;                     // global pixel (n*hw + p): consecutive threads, one plane
    const int q = (int)(u / npix);
    const int64_t n = gp / hw, p = gp - n * hw;
    const float* src = in + gp * c;
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c0 = q * 8 + 2 * j, c1 = c0 + 1;
      const float f0 = c0 < c ? src[c0] : 0.0f;
      const float f1 = c1 < c ? src[c1] : 0.0f;
      __nv_bfloat162 v = __floats2bfloat162_rn(f0, f1);
      w[j] = *reinterpret_cast<uint32_t*>(&v);
    }
    *reinterpret_cast<uint4*>(out + ((n * planes + q) * hw + p) * 8) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

__global__ void k_init(int* counts, int n, int* orig, int32_t* path, float* margin, int nmax) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) counts[0] = n;
  if (i < n) {
    orig[i] = i;
    if (path) path[i] = 0;
    if (margin) margin[i] = __int_as_float(0x7f800000);   // +inf: no predicate evaluated yet
  }
}

// ------------------------------------------------------- a2 + a3 head/predicate
constexpr int HEAD_THREADS = 256;

__global__ void __launch_bounds__(HEAD_THREADS) k_head(const HeadArgs a) {
  extern __shared__ float sh[];
  float* part = sh;                                // [HEAD_THREADS][8]
  float* g = part + HEAD_THREADS * 8;              // [C]
  float* z = g + a.C;                              // [K]
  __shared__ float red[HEAD_THREADS / 32];
  const int n_live = *a.n_live;
  const int t = threadIdx.x;
  const int G = a.C / 8;                           // 16-byte channel groups per pixel
  const int P = HEAD_THREADS / G;                  // pixel stride
  for (int row = blockIdx.x; row < n_live; row += gridDim.x) {
    const uint16_t* h = a.h + (size_t)row * a.HW * a.C;
    // GAP: thread (p0, grp) sums its 8 channels over pixels p0, p0+P, ...
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (a.pooled) {                                // fused into the producing block: just load
      for (int c = t; c < a.C; c += HEAD_THREADS) g[c] = a.pooled[(size_t)row * a.C + c];
    } else if (t < G * P) {
      const int grp = t % G;
      if (a.h32 && a.h32_pair) {
        // pair stream: value = bf16 hi (the NHWC operand copy) + bf16 lo
        const uint16_t* lo = reinterpret_cast<const uint16_t*>(a.h32) + (size_t)row * a.HW * a.C;
        for (int p = t / G; p < a.HW; p += P) {
          const uint4 vh = __ldg(reinterpret_cast<const uint4*>(h + (size_t)p * a.C + grp * 8));
          const uint4 vl = __ldg(reinterpret_cast<const uint4*>(lo + (size_t)p * a.C + grp * 8));
          const uint32_t uh[4] = {vh.x, vh.y, vh.z, vh.w}, ul[4] = {vl.x, vl.y, vl.z, vl.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            acc[2 * j] += __uint_as_float(uh[j] << 16) + __uint_as_float(ul[j] << 16);
            acc[2 * j + 1] += __uint_as_float(uh[j] & 0xFFFF0000u) + __uint_as_float(ul[j] & 0xFFFF0000u);
          }
        }
      } else if (a.h32) {
        const float* h32 = a.h32 + (size_t)row * a.HW * a.C;
        for (int p = t / G; p < a.HW; p += P) {
          const float4* q = reinterpret_cast<const float4*>(h32 + (size_t)p * a.C + grp * 8);
          const float4 v0 = __ldg(q), v1 = __ldg(q + 1);
          acc[0] += v0.x; acc[1] += v0.y; acc[2] += v0.z; acc[3] += v0.w;
          acc[4] += v1.x; acc[5] += v1.y; acc[6] += v1.z; acc[7] += v1.w;
        }
      } else {
        // bf16 channel-planar [C/8][HW][8] (or NHWC [HW][C])
        for (int p = t / G; p < a.HW; p += P) {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(a.nhwc ? h + (size_t)p * a.C + grp * 8
                                                                      : h + ((size_t)grp * a.HW + p) * 8));
          const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            acc[2 * j] += __uint_as_float(u[j] << 16);
            acc[2 * j + 1] += __uint_as_float(u[j] & 0xFFFF0000u);
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) part[t * 8 + j] = acc[j];
    __syncthreads();
    for (int c = t; c < a.C && !a.pooled; c += HEAD_THREADS) {
      const int grp = c >> 3, j = c & 7;
      float s = 0.0f;
      for (int q = 0; q < P; ++q) s += part[(q * G + grp) * 8 + j];
      g[c] = s / (float)a.HW;
      if (a.wt) a.gpool[(size_t)row * a.C + c] = g[c];
      if (a.pooled_out) a.pooled_out[(size_t)row * a.C + c] = g[c];
    }
    __syncthreads();
    if (a.wt) continue;                            // wide head: FC + predicate in k_head_fc
    // FC: one warp per output row, lanes over channels, fixed shuffle tree.
    const int warp = t >> 5, lane = t & 31;
    for (int j = warp; j < a.K; j += HEAD_THREADS / 32) {
      const uint16_t* wr = a.w + (size_t)j * a.C;
      float s = 0.0f;
      for (int c = lane; c < a.C; c += 32) s += bf16f(wr[c]) * g[c];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) z[j] = s + a.b[j];
    }
    __syncthreads();
    for (int j = t; j < a.K; j += HEAD_THREADS) a.z[(size_t)row * a.K + j] = z[j];
    // predicate
    if (a.kind == 0) {
      float m = -INFINITY;
      for (int j = t; j < a.K; j += HEAD_THREADS) m = fmaxf(m, z[j]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) red[warp] = m;
      __syncthreads();
      m = red[0];
      for (int w = 1; w < HEAD_THREADS / 32; ++w) m = fmaxf(m, red[w]);
      __syncthreads();
      float s = 0.0f;
      for (int j = t; j < a.K; j += HEAD_THREADS) s += expf(z[j] - m);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) red[warp] = s;
      __syncthreads();
      if (t == 0) {
        float tot = 0.0f;
        for (int w = 0; w < HEAD_THREADS / 32; ++w) tot += red[w];
        const float conf = 1.0f / tot;           // max_j softmax(z)_j
        a.flag[row] = conf >= a.thr ? 1 : 0;     // reading R1: conf >= tau exits
        if (a.pred) a.pred[row] = conf;
      }
    } else if (t == 0) {
      if (a.kind == 1) {
        const float p = 1.0f / (1.0f + expf(-z[0]));
        a.flag[row] = p > a.thr ? 1 : 0;         // reading R2: p > thr executes
        if (a.pred) a.pred[row] = p;
      } else {
        a.flag[row] = 1;
        if (a.pred) a.pred[row] = 1.0f;
      }
    }
    __syncthreads();
  }
}

// Head on fused-GAP features (a.pooled) with K <= 32, C <= 64: one warp per live row, lane k
// computes logit k (sum over c ascending), then the predicate with warp reductions.
__global__ void __launch_bounds__(256) k_head_small(const HeadArgs a) {
  const int n_live = *a.n_live;
  const int lane = threadIdx.x & 31;
  for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < n_live; row += (gridDim.x * blockDim.x) >> 5) {
    const float* gp = a.pooled + (size_t)row * a.C;
    const float g0 = lane < a.C ? gp[lane] : 0.f, g1 = lane + 32 < a.C ? gp[lane + 32] : 0.f;
    float z = -INFINITY;
    if (lane < a.K) {
      const uint16_t* wr = a.w + (size_t)lane * a.C;
      float sacc = 0.f;
      for (int c = 0; c < a.C; ++c) {
        const float gc = __shfl_sync(0xffffffffu, c < 32 ? g0 : g1, c & 31);
        sacc += bf16f(wr[c]) * gc;
      }
      z = sacc + a.b[lane];
      a.z[(size_t)row * a.K + lane] = z;
    } else {
      for (int c = 0; c < a.C; ++c) (void)__shfl_sync(0xffffffffu, c < 32 ? g0 : g1, c & 31);
    }
    if (a.kind == 0) {
      float m = z;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      float e = lane < a.K ? expf(z - m) : 0.f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
      if (lane == 0) {
        const float conf = 1.0f / e;               // max_j softmax(z)_j
        a.flag[row] = conf >= a.thr ? 1 : 0;       // reading R1: conf >= tau exits
        if (a.pred) a.pred[row] = conf;
      }
    } else if (lane == 0) {
      if (a.kind == 1) {
        const float pr = 1.0f / (1.0f + expf(-z));
        a.flag[row] = pr > a.thr ? 1 : 0;          // reading R2: p > thr executes
        if (a.pred) a.pred[row] = pr;
      } else {
        a.flag[row] = 1;
        if (a.pred) a.pred[row] = 1.0f;
      }
    }
  }
}

// Wide heads (K = 1000): logits for FC_ROWS samples x 256 classes per CTA from the pooled
// features, so the [C][K] weights stream once per FC_ROWS samples (the per-sample form re-read
// 4 MB of weights per ResNet-50 sample).  Thread = one class; the pooled rows sit in SMEM as
// [C][FC_ROWS] (two LDS.128 per c, broadcast); the sum over c runs in order, fp32.
constexpr int FC_ROWS = 8;
constexpr int FC_UNROLL = 8;

__global__ void __launch_bounds__(HEAD_THREADS) k_head_fc(const HeadArgs a) {
  extern __shared__ float gs[];                    // [C][FC_ROWS]
  const int n_live = *a.n_live;
  const int t = threadIdx.x;
  const int j = blockIdx.y * HEAD_THREADS + t;     // class
  for (int r0 = blockIdx.x * FC_ROWS; r0 < n_live; r0 += gridDim.x * FC_ROWS) {
    const int nr = min(FC_ROWS, n_live - r0);
    for (int i = t; i < FC_ROWS * a.C; i += HEAD_THREADS) {
      const int r = i / a.C, c = i - r * a.C;
      gs[c * FC_ROWS + r] = r < nr ? a.gpool[(size_t)(r0 + r) * a.C + c] : 0.0f;
    }
    __syncthreads();
    float acc[FC_ROWS];
#pragma unroll
    for (int r = 0; r < FC_ROWS; ++r) acc[r] = 0.0f;
    if (j < a.K) {
      const uint16_t* wj = a.wt + j;
      for (int c0 = 0; c0 < a.C; c0 += FC_UNROLL) {
        float w[FC_UNROLL];
#pragma unroll
        for (int u = 0; u < FC_UNROLL; ++u) w[u] = bf16f(__ldg(wj + (size_t)(c0 + u) * a.K));
#pragma unroll
        for (int u = 0; u < FC_UNROLL; ++u) {
          const float4 g0 = *reinterpret_cast<const float4*>(gs + (c0 + u) * FC_ROWS);
          const float4 g1 = *reinterpret_cast<const float4*>(gs + (c0 + u) * FC_ROWS + 4);
          acc[0] = fmaf(w[u], g0.x, acc[0]); acc[1] = fmaf(w[u], g0.y, acc[1]);
          acc[2] = fmaf(w[u], g0.z, acc[2]); acc[3] = fmaf(w[u], g0.w, acc[3]);
          acc[4] = fmaf(w[u], g1.x, acc[4]); acc[5] = fmaf(w[u], g1.y, acc[5]);
          acc[6] = fmaf(w[u], g1.z, acc[6]); acc[7] = fmaf(w[u], g1.w, acc[7]);
        }
      }
      const float bj = a.b[j];
      for (int r = 0; r < nr; ++r) a.z[(size_t)(r0 + r) * a.K + j] = acc[r] + bj;
    }
    __syncthreads();
  }
}

// Predicate of a wide head: one warp per live row over the logits in a.z (fixed-order reductions).
__global__ void k_head_pred(const HeadArgs a) {
  const int n_live = *a.n_live;
  const int lane = threadIdx.x & 31;
  for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < n_live; row += (gridDim.x * blockDim.x) >> 5) {
    const float* z = a.z + (size_t)row * a.K;
    float m = -INFINITY;
    for (int j = lane; j < a.K; j += 32) m = fmaxf(m, z[j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float sum = 0.0f;
    for (int j = lane; j < a.K; j += 32) sum += expf(z[j] - m);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) {
      if (a.kind == 0) {
        const float conf = 1.0f / sum;             // max_j softmax(z)_j
        a.flag[row] = conf >= a.thr ? 1 : 0;       // reading R1: conf >= tau exits
        if (a.pred) a.pred[row] = conf;
      } else {
        a.flag[row] = 1;                           // final head
        if (a.pred) a.pred[row] = 1.0f;
      }
    }
  }
}

// Wide head operand: pooled fp32 features [n][C] -> the split bf16 pair [hi | lo] per row
// ([n][2C]; hi = bf16_rn(g), lo = bf16_rn(g - hi)), the A operand of the tensor-core head GEMM.
__global__ void k_pool_split(const float* __restrict__ g, uint16_t* __restrict__ a2, const int* n_live, int C) {
  const int n = *n_live;
  const int C4 = C >> 2;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)n * C4;
       i += (long long)gridDim.x * blockDim.x) {
    const long long row = i / C4;
    const int c = (int)(i - row * C4) * 4;
    const float4 v = __ldg(reinterpret_cast<const float4*>(g + row * C + c));
    const uint32_t h01 = pack_bf16x2_rn(v.x, v.y), h23 = pack_bf16x2_rn(v.z, v.w);
    const uint32_t l01 = pack_bf16x2_rn(v.x - __uint_as_float(h01 << 16), v.y - __uint_as_float(h01 & 0xFFFF0000u));
    const uint32_t l23 = pack_bf16x2_rn(v.z - __uint_as_float(h23 << 16), v.w - __uint_as_float(h23 & 0xFFFF0000u));
    uint16_t* r = a2 + row * 2 * C;
    *reinterpret_cast<uint2*>(r + c) = make_uint2(h01, h23);
    *reinterpret_cast<uint2*>(r + C + c) = make_uint2(l01, l23);
  }
}

// Recurrent gate: one warp per live row.  Lane j < 4H (two passes of 32 lanes) computes the
// pre-activation of gate row j in a fixed order (b_ih + b_hh, then w_ih . u ascending, then
// w_hh . h ascending); lanes k < H then update c_k, h_k from rows (k, H+k, 2H+k, 3H+k).
__global__ void k_rnn_gate(const RnnGateArgs a) {
  const int n_live = *a.n_live;
  const int lane = threadIdx.x & 31;
  const int H = a.hidden, NI = a.n_in, H4 = 4 * H;
  const float* w_ih = a.w;
  const float* w_hh = w_ih + (size_t)H4 * NI;
  const float* b_ih = w_hh + (size_t)H4 * H;
  const float* b_hh = b_ih + H4;
  for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < n_live; row += (gridDim.x * blockDim.x) >> 5) {
    float* st = a.state + (size_t)a.orig[row] * 2 * H;
    const float uv = lane < NI ? a.u[(size_t)row * a.u_stride + lane] : 0.f;
    const float hv = lane < H ? st[lane] : 0.f;
    const float cv = lane < H ? st[H + lane] : 0.f;
    float pre[2];
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
      const int j = lane + 32 * pass;
      float acc = 0.f;
      if (j < H4) acc = b_ih[j] + b_hh[j];
      for (int k = 0; k < NI; ++k) {
        const float uk = __shfl_sync(0xffffffffu, uv, k);
        if (j < H4) acc = fmaf(w_ih[(size_t)j * NI + k], uk, acc);
      }
      for (int k = 0; k < H; ++k) {
        const float hk = __shfl_sync(0xffffffffu, hv, k);
        if (j < H4) acc = fmaf(w_hh[(size_t)j * H + k], hk, acc);
      }
      pre[pass] = acc;
    }
    // gate row j lives in lane j % 32 of pass j / 32
    auto fetch = [&](int j) {
      const float v0 = __shfl_sync(0xffffffffu, pre[0], j & 31);
      const float v1 = __shfl_sync(0xffffffffu, pre[1], j & 31);
      return j < 32 ? v0 : v1;
    };
    const int k = lane < H ? lane : 0;
    const float gi = fetch(k), gf = fetch(H + k), gg = fetch(2 * H + k), go = fetch(3 * H + k);
    const float i_ = 1.f / (1.f + expf(-gi)), f_ = 1.f / (1.f + expf(-gf));
    const float g_ = tanhf(gg), o_ = 1.f / (1.f + expf(-go));
    const float c2 = f_ * cv + i_ * g_;
    const float h2 = o_ * tanhf(c2);
    float zc = lane < H ? a.w_out[lane] * h2 : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) zc += __shfl_xor_sync(0xffffffffu, zc, o);
    if (lane < H) {
      st[lane] = h2;
      st[H + lane] = c2;
    }
    if (lane == 0) {
      const float p = 1.0f / (1.0f + expf(-(zc + a.b_out)));
      a.flag[row] = p > a.thr ? 1 : 0;           // reading R2: p > thr executes
      if (a.pred) a.pred[row] = p;
    }
  }
}


// ------------------------------------------------------------ a4 compaction
constexpr int CMP_THREADS = 1024;

__global__ void __launch_bounds__(CMP_THREADS) k_compact(const uint8_t* __restrict__ flag, const int* n_live,
                                                         const int* __restrict__ orig, int* list1, int* list0,
                                                         int* counts_out, int* orig_next, int mode, int32_t* path,
                                                         int32_t path_bit, const float* __restrict__ pred, float thr,
                                                         float* margin) {
  __shared__ int wsum[CMP_THREADS / 32];
  __shared__ int total1_s;
  ptx::pdl_wait();
  ptx::pdl_trigger();
  const int n = *n_live;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int ipt = (n + CMP_THREADS - 1) / CMP_THREADS;
  const int b = min(n, t * ipt), e = min(n, b + ipt);
  // up to CMP_IPT rows per thread: flags / orig ids loaded once, unrolled (independent loads)
  constexpr int CMP_IPT = 8;
  const bool fast = ipt <= CMP_IPT;
  uint8_t fr[CMP_IPT];
  int orr[CMP_IPT];
  int c1 = 0;
  if (fast) {
#pragma unroll
    for (int k = 0; k < CMP_IPT; ++k) {
      fr[k] = b + k < e ? flag[b + k] : 0;
      orr[k] = b + k < e ? orig[b + k] : 0;
      c1 += fr[k] != 0;
    }
  } else {
    for (int i = b; i < e; ++i) c1 += flag[i] != 0;
  }
  // block-wide exclusive scan of c1 (warp shuffles, then warp totals)
  int x = c1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int v = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    wsum[lane] = v;                              // inclusive warp-total prefix
    if (lane == 31) total1_s = v;
  }
  __syncthreads();
  const int excl = x - c1 + (warp > 0 ? wsum[warp - 1] : 0);
  const int total1 = total1_s;
  int o1 = excl;                                 // flag==1 rows before my chunk
  int o0 = b - excl;                             // flag==0 rows before my chunk
  if (fast) {
#pragma unroll
    for (int k = 0; k < CMP_IPT; ++k) {
      if (b + k >= e) break;
      const int i = b + k, oi = orr[k];
      if (margin) margin[oi] = fminf(margin[oi], fabsf(pred[i] - thr));   // per-sample min |pred - thr|
      if (fr[k]) {
        list1[o1] = i;
        if (mode == 1) {
          orig_next[o1] = oi;
          path[oi] |= path_bit;
        }
        ++o1;
      } else {
        list0[o0] = i;
        orig_next[(mode == 1 ? total1 : 0) + o0] = oi;
        ++o0;
      }
    }
  }
  for (int i = fast ? e : b; i < e; ++i) {
    const int oi = orig[i];
    if (margin) margin[oi] = fminf(margin[oi], fabsf(pred[i] - thr));
    if (flag[i]) {
      list1[o1] = i;
      if (mode == 1) {
        orig_next[o1] = oi;
        path[oi] |= path_bit;
      }
      ++o1;
    } else {
      list0[o0] = i;
      orig_next[(mode == 1 ? total1 : 0) + o0] = oi;
      ++o0;
    }
  }
  if (t == 0) {
    counts_out[0] = total1;
    counts_out[1] = n - total1;
  }
}

// ---------------------------------------------------------------- a6 scatter
__global__ void k_scatter(const float* __restrict__ z, int K, const int* __restrict__ list, const int* count,
                          const int* __restrict__ orig, float* out_logits, int32_t* out_path, int32_t path_val) {
  const int cnt = *count;
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int j = blockIdx.x * wpb + (threadIdx.x >> 5); j < cnt; j += gridDim.x * wpb) {
    const int i = list[j];
    const int o = orig[i];
    for (int c = lane; c < K; c += 32) out_logits[(size_t)o * K + c] = z[(size_t)i * K + c];
    if (lane == 0 && path_val >= 0) out_path[o] = path_val;
  }
}

// ----------------------------------------------------------------- a5 gather
__global__ void __launch_bounds__(256) k_gather(const GatherArgs a) {
  const int cnt = *a.count;
  const int off = a.dst_off_count ? *a.dst_off_count : 0;
  const int epu = 16 / a.elem_bytes;             // elements per 16-byte unit
  const int64_t U = a.row_elems_dst / epu;       // 16-byte units per destination row
  const int64_t Us = a.row_elems_src / epu;
  const int64_t total = (int64_t)cnt * U;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint4* src = reinterpret_cast<const uint4*>(a.src);
  uint4* dst = reinterpret_cast<uint4*>(a.dst);
  if (a.mode == 0) {
    for (int64_t u0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u0 < total; u0 += 4 * stride) {
      uint4 v[4];
      int64_t di[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t u = u0 + k * stride;
        di[k] = -1;
        if (u < total) {
          const int64_t j = u / U, q = u - j * U;
          v[k] = __ldg(src + (int64_t)a.list[j] * Us + q);
          di[k] = (off + j) * U + q;
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (di[k] >= 0) dst[di[k]] = v[k];
    }
  } else if (a.elem_bytes == 2 && a.dst_nhwc) {
    // option A, bf16 channel-planar src [C/8][H][W][8] -> NHWC dst [H/2][W/2][2C] (2C % 64 == 0)
    const int Wo = a.W / 2, gpp = 2 * a.C / 8, pad = a.C / 2;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total; u += stride) {
      const int64_t j = u / U;
      const int64_t r = u - j * U;
      const int p = (int)(r / gpp), q = (int)(r - (int64_t)p * gpp);
      const int ho = p / Wo, wo = p - ho * Wo;
      const int cs = q * 8 - pad;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (cs >= 0 && cs < a.C) {
        const int64_t e = (int64_t)a.list[j] * a.row_elems_src + ((int64_t)(cs / 8) * a.H * a.W + (2 * ho) * a.W + 2 * wo) * 8;
        v = __ldg(src + e / 8);
      }
      dst[(off + j) * U + r] = v;
    }
  } else if (a.elem_bytes == 2) {
    // option A, bf16 channel-planar: dst [2C/8][H/2][W/2][8] from src [C/8][H][W][8]
    const int Ho = a.H / 2, Wo = a.W / 2, HWo = Ho * Wo, padp = a.C / 16;   // C/2 channels = C/16 planes
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total; u += stride) {
      const int64_t j = u / U;
      const int64_t r = u - j * U;
      const int pd = (int)(r / HWo), p = (int)(r - (int64_t)pd * HWo);
      const int ho = p / Wo, wo = p - ho * Wo;
      const int ps = pd - padp;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (ps >= 0 && ps < a.C / 8) {
        const int64_t e = (int64_t)a.list[j] * a.row_elems_src + ((int64_t)ps * a.H * a.W + (2 * ho) * a.W + 2 * wo) * 8;
        v = __ldg(src + e / 8);
      }
      dst[(off + j) * U + r] = v;
    }
  } else {
    // option A, fp32 NHWC: dst [H/2][W/2][2C] from src [H][W][C]: pixel (2ho, 2wo), channel c - C/2
    const int Wo = a.W / 2, Cd = 2 * a.C, qpp = Cd / epu, pad = a.C / 2;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total; u += stride) {
      const int64_t j = u / U;
      const int64_t r = u - j * U;
      const int p = (int)(r / qpp), q = (int)(r - (int64_t)p * qpp);
      const int ho = p / Wo, wo = p - ho * Wo;
      const int cs = q * epu - pad;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (cs >= 0 && cs < a.C) {
        const int64_t e = (int64_t)a.list[j] * a.row_elems_src + ((int64_t)(2 * ho) * a.W + 2 * wo) * a.C + cs;
        v = __ldg(src + e / epu);
      }
      dst[(off + j) * U + r] = v;
    }
  }
}

// ------------------------------------------------------------------ max pool
// one thread per (sample, output pixel, 8-channel group); consecutive threads =
// consecutive output pixels of one group (planar stores coalesce).
__global__ void k_maxpool(const PoolArgs a) {
  const int n_live = *a.n_live;
  const int G = a.C / 8;
  const int HWo = a.Ho * a.Wo;
  const int64_t total = (int64_t)n_live * G * HWo;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total; u += (int64_t)gridDim.x * blockDim.x) {
    int p, g;
    int64_t n;
    if (a.nhwc) {                                    // consecutive threads = consecutive channel groups
      g = (int)(u % G);
      const int64_t t = u / G;
      p = (int)(t % HWo);
      n = t / HWo;
    } else {
      p = (int)(u % HWo);
      const int64_t t = u / HWo;
      g = (int)(t % G);
      n = t / G;
    }
    const int ho = p / a.Wo, wo = p - (p / a.Wo) * a.Wo;
    float m[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) m[j] = -INFINITY;
    for (int r = 0; r < a.k; ++r) {
      const int hi = ho * a.stride - a.pad + r;
      if (hi < 0 || hi >= a.H) continue;
      for (int s2 = 0; s2 < a.k; ++s2) {
        const int wi = wo * a.stride - a.pad + s2;
        if (wi < 0 || wi >= a.W) continue;
        const int64_t pix = (int64_t)hi * a.W + wi;
        if (a.x32) {
          const float4* q = reinterpret_cast<const float4*>(a.x32 + (n * a.H * a.W + pix) * a.C + g * 8);
          const float4 v0 = __ldg(q), v1 = __ldg(q + 1);
          m[0] = fmaxf(m[0], v0.x); m[1] = fmaxf(m[1], v0.y); m[2] = fmaxf(m[2], v0.z); m[3] = fmaxf(m[3], v0.w);
          m[4] = fmaxf(m[4], v1.x); m[5] = fmaxf(m[5], v1.y); m[6] = fmaxf(m[6], v1.z); m[7] = fmaxf(m[7], v1.w);
        } else {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(
              a.nhwc ? a.x + (n * a.H * a.W + pix) * a.C + g * 8 : a.x + ((n * G + g) * (int64_t)a.H * a.W + pix) * 8));
          const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            m[2 * j] = fmaxf(m[2 * j], __uint_as_float(w4[j] << 16));
            m[2 * j + 1] = fmaxf(m[2 * j + 1], __uint_as_float(w4[j] & 0xFFFF0000u));
          }
        }
      }
    }
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      __nv_bfloat162 v = __floats2bfloat162_rn(m[2 * j], m[2 * j + 1]);
      o[j] = *reinterpret_cast<uint32_t*>(&v);
    }
    *reinterpret_cast<uint4*>(a.nhwc ? a.y + (n * HWo + p) * a.C + g * 8 : a.y + ((n * G + g) * (int64_t)HWo + p) * 8) =
        make_uint4(o[0], o[1], o[2], o[3]);
    if (a.y32) {
      float4* q = reinterpret_cast<float4*>(a.y32 + (n * HWo + p) * a.C + g * 8);
      q[0] = make_float4(m[0], m[1], m[2], m[3]);
      q[1] = make_float4(m[4], m[5], m[6], m[7]);
    }
  }
}

// 3x3 / stride-2 / pad-1 max pool over the space-to-depth stem output: input [n][Ho][Wo][4C],
// channel (b*2+b')*C + c holds pixel (2P+b, 2Q+b'); output pixel (P, Q) takes the max over
// rows 2P-1..2P+1 x cols 2Q-1..2Q+1 = its own 4 phases, phases b = 1 of block P-1, b' = 1 of
// block Q-1 and phase (1,1) of block (P-1, Q-1).  One thread per (sample, pixel, 8-channel group).
__global__ void k_maxpool_s2d(const PoolArgs a) {
  // grid: x over (pixel, group) items of one sample, y over samples; 32-bit index math (the
  // 64-bit divisions of a flat index made this kernel ALU-bound)
  const int n_live = *a.n_live;
  const int G = a.C / 8, C4 = 4 * a.C;
  const int items = a.Ho * a.Wo * G;
  for (int n = blockIdx.y; n < n_live; n += gridDim.y) {
    const uint16_t* xs = a.x + (size_t)n * a.Ho * a.Wo * C4;
    uint16_t* ys = a.y + (size_t)n * a.Ho * a.Wo * a.C;
    for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < items; w += gridDim.x * blockDim.x) {
      const int p = w / G, g = w - (w / G) * G;
      const int P = p / a.Wo, Q = p - (p / a.Wo) * a.Wo;
      float m[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) m[j] = -INFINITY;
      auto take = [&](int pp, int qq, int ph) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(xs + (pp * a.Wo + qq) * C4 + ph * a.C + g * 8));
        const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          m[2 * j] = fmaxf(m[2 * j], __uint_as_float(w4[j] << 16));
          m[2 * j + 1] = fmaxf(m[2 * j + 1], __uint_as_float(w4[j] & 0xFFFF0000u));
        }
      };
#pragma unroll
      for (int ph = 0; ph < 4; ++ph) take(P, Q, ph);
      if (P > 0) { take(P - 1, Q, 2); take(P - 1, Q, 3); }
      if (Q > 0) { take(P, Q - 1, 1); take(P, Q - 1, 3); }
      if (P > 0 && Q > 0) take(P - 1, Q - 1, 3);
      uint32_t o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        __nv_bfloat162 v = __floats2bfloat162_rn(m[2 * j], m[2 * j + 1]);
        o[j] = *reinterpret_cast<uint32_t*>(&v);
      }
      *reinterpret_cast<uint4*>(ys + (size_t)p * a.C + g * 8) = make_uint4(o[0], o[1], o[2], o[3]);
      if (a.y32) {
        float4* q = reinterpret_cast<float4*>(a.y32 + ((size_t)n * a.Ho * a.Wo + p) * a.C + g * 8);
        q[0] = make_float4(m[0], m[1], m[2], m[3]);
        q[1] = make_float4(m[4], m[5], m[6], m[7]);
      }
    }
  }
}

// fp32 NHWC [n][H][W][c] -> bf16 4x4 space-to-depth [n][H/4][W/4][64]; one thread per output
// pixel: the 4 input rows of its block are 4 contiguous runs of 4*c floats (c == 3: 3 float4
// each; lanes = consecutive blocks, so a warp reads contiguous 1.5 KB rows), 128 B out.
// a0, 2x2 space-to-depth: thread per output block (32-bit index math: the launcher bounds the
// block count); channel (dy*2+dx)*c + ci, zeros up to 16
__global__ void k_cast_s2d2(const float* __restrict__ in, uint16_t* __restrict__ out, int64_t total, int H, int W,
                            int c) {
  const uint32_t Wb = (uint32_t)(W / 2), Hb = (uint32_t)(H / 2);
  for (uint32_t blk = blockIdx.x * blockDim.x + threadIdx.x; blk < (uint32_t)total; blk += gridDim.x * blockDim.x) {
    const uint32_t t = blk / Wb, Q = blk - t * Wb;
    const uint32_t n = t / Hb, Pr = t - n * Hb;
    float v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = 0.0f;
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx)
        for (int ci = 0; ci < c; ++ci)
          v[(dy * 2 + dx) * c + ci] =
              __ldg(in + (((size_t)n * H + 2 * Pr + dy) * (size_t)W + 2 * Q + dx) * c + ci);
    uint4* dst = reinterpret_cast<uint4*>(out + (size_t)blk * 16);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      uint32_t o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        __nv_bfloat162 b = __floats2bfloat162_rn(v[8 * j + 2 * k], v[8 * j + 2 * k + 1]);
        o[k] = *reinterpret_cast<uint32_t*>(&b);
      }
      dst[j] = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

__global__ void __launch_bounds__(256) k_cast_s4d(const float* __restrict__ in, uint16_t* __restrict__ out,
                                                   int64_t total, int H, int W, int c, int vec) {
  // a warp converts 32 consecutive output pixels (4 KB of output) and stores them through SMEM
  // as contiguous 512-byte rows (direct 16-byte stores at a 128-byte lane stride left the
  // kernel at ~3.4 TB/s)
  __shared__ uint4 stage[8][256];
  const int Wb = W / 4, Hb = H / 4;
  const int lane = threadIdx.x & 31;
  uint4* sw = stage[threadIdx.x >> 5];
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); base < total;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pix = base + lane;
    const bool ok = pix < total;
    // 32-bit index arithmetic when the launch fits (64-bit division is a long software sequence)
    int Q, P;
    int64_t n;
    if (total < (int64_t)1 << 31) {
      const uint32_t p32 = (uint32_t)pix, t32 = p32 / (uint32_t)Wb;
      Q = (int)(p32 - t32 * (uint32_t)Wb);
      const uint32_t n32 = t32 / (uint32_t)Hb;
      P = (int)(t32 - n32 * (uint32_t)Hb);
      n = n32;
    } else {
      Q = (int)(pix % Wb);
      const int64_t t = pix / Wb;
      P = (int)(t % Hb);
      n = t / Hb;
    }
    float v[64];
#pragma unroll
    for (int k = 0; k < 64; ++k) v[k] = 0.0f;
    if (ok && vec) {
#pragma unroll
      for (int pr = 0; pr < 4; ++pr) {
        const float4* src = reinterpret_cast<const float4*>(in + ((n * H + 4 * P + pr) * (int64_t)W + 4 * Q) * 3);
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const float4 f = __ldg(src + q);
          v[pr * 12 + 4 * q] = f.x; v[pr * 12 + 4 * q + 1] = f.y; v[pr * 12 + 4 * q + 2] = f.z; v[pr * 12 + 4 * q + 3] = f.w;
        }
      }
    } else if (ok) {
      for (int ch = 0; ch < 16 * c; ++ch) {
        const int ph = ch / c, ci = ch - ph * c;
        v[ch] = __ldg(in + ((n * H + 4 * P + (ph >> 2)) * (int64_t)W + 4 * Q + (ph & 3)) * c + ci);
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        __nv_bfloat162 b = __floats2bfloat162_rn(v[8 * j + 2 * k], v[8 * j + 2 * k + 1]);
        o[k] = *reinterpret_cast<uint32_t*>(&b);
      }
      sw[lane * 8 + (j ^ (lane & 7))] = make_uint4(o[0], o[1], o[2], o[3]);   // XOR: conflict-free
    }
    __syncwarp();
    uint4* dst = reinterpret_cast<uint4*>(out + base * 64);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int e = k * 32 + lane, pe = e >> 3;
      if (base + pe < total) dst[e] = sw[pe * 8 + ((e & 7) ^ (pe & 7))];
    }
    __syncwarp();
  }
}

__global__ void k_gap_reduce(const float* __restrict__ part, int G, float* __restrict__ pooled, const int* n_live,
                             int HW, int C) {
  const int n_rows = *n_live;
  const int64_t total = (int64_t)n_rows * C;
  const int ng = HW / G;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total; u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = u / C;
    const int c = (int)(u - n * C);
    const float* p = part + (size_t)n * ng * C + c;
    float sum = 0.f;                                 // fixed order: groups k = 0, 1, ... of sample n
    for (int k = 0; k < ng; ++k) sum += p[(size_t)k * C];
    pooled[n * C + c] = sum / (float)HW;
  }
}

}  // namespace

cudaError_t launch_gap_reduce(const float* gap_part, int G, float* pooled, const int* n_live, int max_rows, int HW, int C,
                              cudaStream_t s) {
  if (G < 1 || HW % G) return cudaErrorInvalidValue;
  int64_t blocks = ((int64_t)max_rows * C + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  k_gap_reduce<<<(int)blocks, 256, 0, s>>>(gap_part, G, pooled, n_live, HW, C);
  return cudaGetLastError();
}

cudaError_t launch_cast_s2d2(const float* in, uint16_t* out, int64_t n, int H, int W, int c, cudaStream_t s) {
  if (H % 2 || W % 2 || c > 4 || n * (H / 2) * (W / 2) >= ((int64_t)1 << 31)) return cudaErrorInvalidValue;
  const int64_t total = n * (H / 2) * (W / 2);
  if (total == 0) return cudaSuccess;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  k_cast_s2d2<<<(int)blocks, 256, 0, s>>>(in, out, total, H, W, c);
  return cudaGetLastError();
}

cudaError_t launch_cast_s4d(const float* in, uint16_t* out, int64_t n, int H, int W, int c, cudaStream_t s) {
  if (H % 4 || W % 4 || c > 4) return cudaErrorInvalidValue;
  const int64_t total = n * (H / 4) * (W / 4);
  if (total == 0) return cudaSuccess;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  const int vec = c == 3 && ((uintptr_t)in & 15) == 0;
  k_cast_s4d<<<(int)blocks, 256, 0, s>>>(in, out, total, H, W, c, vec);
  return cudaGetLastError();
}

cudaError_t launch_maxpool(const PoolArgs& a, int max_rows, int num_sms, cudaStream_t s) {
  if (a.s2d) {
    if (!a.nhwc || a.k != 3 || a.stride != 2 || a.pad != 1) return cudaErrorInvalidValue;
    const int items = (a.C / 8) * a.Ho * a.Wo;
    const int bx = (items + 255) / 256;
    const int by = max_rows < 1 ? 1 : max_rows > 65535 ? 65535 : max_rows;
    k_maxpool_s2d<<<dim3(bx, by), 256, 0, s>>>(a);
    return cudaGetLastError();
  }
  const int64_t total = (int64_t)max_rows * (a.C / 8) * a.Ho * a.Wo;
  int64_t blocks = (total + 255) / 256;
  if (blocks > (int64_t)num_sms * 16) blocks = (int64_t)num_sms * 16;
  if (blocks < 1) blocks = 1;
  k_maxpool<<<(int)blocks, 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_cast_pad(const float* in, uint16_t* out, int64_t n, int hw, int c, int cp, cudaStream_t s) {
  const int64_t npix = n * hw;
  if (npix == 0) return cudaSuccess;
  int64_t blocks = (npix * (cp / 8) + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_cast_pad<<<(int)blocks, 256, 0, s>>>(in, out, npix, hw, c, cp);
  return cudaGetLastError();
}

cudaError_t launch_init(int* counts, int n, int* orig, int32_t* path, float* margin, int nmax, cudaStream_t s) {
  const int blocks = (n + 255) / 256 > 0 ? (n + 255) / 256 : 1;
  k_init<<<blocks, 256, 0, s>>>(counts, n, orig, path, margin, nmax);
  return cudaGetLastError();
}

// Wide head FC on tcgen05 (k_gemm_tma over the split pair), then the predicate.
static cudaError_t head_fc_tc(const HeadArgs& a, const float* pooled, int max_rows, cudaStream_t s) {
  int gs = (int)(((long long)max_rows * (a.C / 4) + 255) / 256);
  if (gs > a.num_sms * 8) gs = a.num_sms * 8;
  if (gs < 1) gs = 1;
  k_pool_split<<<gs, 256, 0, s>>>(pooled, a.a2, a.n_live, a.C);
  ConvArgs g{};
  g.x = a.a2;
  g.w = a.w2;
  g.bias = a.b2;
  g.y = nullptr;
  g.y32 = a.z;
  g.y32_ld = a.K;
  g.y32_n = a.K;
  g.n_live = a.n_live;
  g.H = g.W = g.Ho = g.Wo = 1;
  g.C = g.K = g.Kp = 2 * a.C;
  g.Cout = a.kpad;
  g.ksz = 1; g.stride = 1; g.pad = 0;
  g.nhwc = g.in_nhwc = 1;
  if (!gemm_tma_eligible(g)) return cudaErrorInvalidValue;
  if (cudaError_t e = launch_gemm_tma(g, max_rows, a.num_sms, s)) return e;
  int gp = (max_rows + 7) / 8;
  if (gp > a.num_sms * 8) gp = a.num_sms * 8;
  if (gp < 1) gp = 1;
  k_head_pred<<<gp, 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_head(const HeadArgs& a, int max_rows, cudaStream_t s) {
  if (a.C % 8 != 0 || a.C / 8 > HEAD_THREADS) return cudaErrorInvalidValue;
  if (a.w2 && a.kind != 1) {                     // wide head, FC on the tensor cores
    if (a.pooled) return head_fc_tc(a, a.pooled, max_rows, s);
    if (!a.gpool || !a.wt) return cudaErrorInvalidValue;
    const size_t smem = (HEAD_THREADS * 8 + a.C + a.K) * sizeof(float);
    if (cudaError_t e = ensure_smem(k_head, smem)) return e;
    int grid = max_rows < a.num_sms * 8 ? max_rows : a.num_sms * 8;
    if (grid < 1) grid = 1;
    k_head<<<grid, HEAD_THREADS, smem, s>>>(a);   // GAP only (a.wt set): pooled -> gpool
    return head_fc_tc(a, a.gpool, max_rows, s);
  }
  if (a.pooled && a.wt) {                        // wide head on pooled features: FC + predicate only
    HeadArgs b = a;
    b.gpool = const_cast<float*>(a.pooled);
    b.pooled = nullptr;
    const size_t smem_fc = (size_t)FC_ROWS * b.C * sizeof(float);
    if (cudaError_t e = ensure_smem(k_head_fc, smem_fc)) return e;
    if (b.kind == 1 || b.C % FC_UNROLL) return cudaErrorInvalidValue;
    int gx = (max_rows + FC_ROWS - 1) / FC_ROWS;
    if (gx > 148 * 2) gx = 148 * 2;
    if (gx < 1) gx = 1;
    k_head_fc<<<dim3(gx, (b.K + HEAD_THREADS - 1) / HEAD_THREADS), HEAD_THREADS, smem_fc, s>>>(b);
    int gp = (max_rows + 7) / 8;
    if (gp > 148 * 8) gp = 148 * 8;
    if (gp < 1) gp = 1;
    k_head_pred<<<gp, 256, 0, s>>>(b);
    return cudaGetLastError();
  }
  if (a.pooled && !a.wt && a.K <= 32 && a.C <= 64) {
    int grid = (max_rows + 7) / 8;
    if (grid > 148 * 16) grid = 148 * 16;
    k_head_small<<<grid > 0 ? grid : 1, 256, 0, s>>>(a);
    return cudaGetLastError();
  }
  const size_t smem = (HEAD_THREADS * 8 + a.C + a.K) * sizeof(float);
  if (cudaError_t e = ensure_smem(k_head, smem)) return e;
  int grid = max_rows < 148 * 8 ? max_rows : 148 * 8;
  if (grid < 1) grid = 1;
  k_head<<<grid, HEAD_THREADS, smem, s>>>(a);
  if (!a.wt) return cudaGetLastError();
  if (a.kind == 1 || !a.gpool) return cudaErrorInvalidValue;
  const size_t smem_fc = (size_t)FC_ROWS * a.C * sizeof(float);
  if (cudaError_t e = ensure_smem(k_head_fc, smem_fc)) return e;
  if (a.C % FC_UNROLL) return cudaErrorInvalidValue;
  int gx = (max_rows + FC_ROWS - 1) / FC_ROWS;
  if (gx > 148 * 2) gx = 148 * 2;
  if (gx < 1) gx = 1;
  k_head_fc<<<dim3(gx, (a.K + HEAD_THREADS - 1) / HEAD_THREADS), HEAD_THREADS, smem_fc, s>>>(a);
  int gp = (max_rows + 7) / 8;
  if (gp > 148 * 8) gp = 148 * 8;
  if (gp < 1) gp = 1;
  k_head_pred<<<gp, 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_rnn_gate(const RnnGateArgs& a, int max_rows, int num_sms, cudaStream_t s) {
  if (a.hidden < 1 || a.hidden > 16 || a.n_in < 1 || a.n_in > 16) return cudaErrorInvalidValue;
  int grid = (max_rows + 7) / 8;
  if (grid > num_sms * 8) grid = num_sms * 8;
  if (grid < 1) grid = 1;
  k_rnn_gate<<<grid, 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_compact(const uint8_t* flag, const int* n_live, const int* orig, int* list1, int* list0,
                           int* counts_out, int* orig_next, int mode, int32_t* path, int32_t path_bit,
                           const float* pred, float thr, float* margin, cudaStream_t s) {
  return launch_k(k_compact, dim3(1), dim3(CMP_THREADS), 0, s, flag, n_live, orig, list1, list0, counts_out, orig_next,
                  mode, path, path_bit, pred, thr, margin);
}

cudaError_t launch_scatter(const float* z, int K, const int* list, const int* count, const int* orig,
                           float* out_logits, int32_t* out_path, int32_t path_val, int max_rows, cudaStream_t s) {
  int blocks = (max_rows + 7) / 8;
  if (blocks > 148 * 4) blocks = 148 * 4;
  if (blocks < 1) blocks = 1;
  k_scatter<<<blocks, 256, 0, s>>>(z, K, list, count, orig, out_logits, out_path, path_val);
  return cudaGetLastError();
}

cudaError_t launch_gather(const GatherArgs& a, int max_rows, int num_sms, cudaStream_t s) {
  const int64_t units = (int64_t)max_rows * (a.row_elems_dst * a.elem_bytes / 16);
  int64_t blocks = (units + 255) / 256;
  if (blocks > (int64_t)num_sms * 8) blocks = (int64_t)num_sms * 8;
  if (blocks < 1) blocks = 1;
  k_gather<<<(int)blocks, 256, 0, s>>>(a);
  return cudaGetLastError();
}

// ------------------------------------------------ a9 survivor rebalancing
// Rows [first, first + n) of the dense survivor tensor leave this rank: record their row ids
// in the run's result space (orig) and their metadata (path word, min margin, global id).
__global__ void k_rb_pack(const int* __restrict__ orig, int first, int n, const int32_t* __restrict__ res_path,
                          const float* __restrict__ res_margin, const long long* __restrict__ ext_gid,
                          long long gid_base, int batch, int* sent_orig, int32_t* meta) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const int o = orig[first + j];
    sent_orig[j] = o;
    const long long gid = o < batch ? gid_base + o : ext_gid[o - batch];
    meta[4 * j + 0] = res_path[o];
    meta[4 * j + 1] = res_margin ? __float_as_int(res_margin[o]) : 0x7f800000;
    meta[4 * j + 2] = (int32_t)(gid & 0xffffffffll);
    meta[4 * j + 3] = (int32_t)(gid >> 32);
  }
}
// Rows received from peers were appended at rows [first, first + n): they get result-space
// ids ext0 + j (past the rank's own rows) and their path word / margin / global id.
__global__ void k_rb_unpack(int* orig, int first, int n, int ext0, int batch, const int32_t* __restrict__ meta,
                            int32_t* res_path, float* res_margin, long long* ext_gid) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const int o = ext0 + j;
    orig[first + j] = o;
    res_path[o] = meta[4 * j + 0];
    if (res_margin) res_margin[o] = __int_as_float(meta[4 * j + 1]);
    ext_gid[o - batch] = (long long)(uint32_t)meta[4 * j + 2] | ((long long)meta[4 * j + 3] << 32);
  }
}
// Results of the rows this rank sent, returned by the reverse plan, scattered home by id.
__global__ void k_rb_return(const int* __restrict__ sent_orig, int n, int K, const float* __restrict__ ret_logits,
                            const int32_t* __restrict__ ret_path, const float* __restrict__ ret_margin,
                            float* res_logits, int32_t* res_path, float* res_margin) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int j = blockIdx.x * wpb + (threadIdx.x >> 5); j < n; j += gridDim.x * wpb) {
    const int o = sent_orig[j];
    for (int c = lane; c < K; c += 32) res_logits[(size_t)o * K + c] = ret_logits[(size_t)j * K + c];
    if (lane == 0) {
      res_path[o] = ret_path[j];
      if (res_margin) res_margin[o] = ret_margin[j];
    }
  }
}
__global__ void k_set_int(int* p, int v) { *p = v; }

cudaError_t launch_rb_pack(const int* orig, int first, int n, const int32_t* res_path, const float* res_margin,
                           const long long* ext_gid, long long gid_base, int batch, int* sent_orig, int32_t* meta,
                           cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  k_rb_pack<<<(n + 255) / 256 < 148 ? (n + 255) / 256 : 148, 256, 0, s>>>(orig, first, n, res_path, res_margin,
                                                                          ext_gid, gid_base, batch, sent_orig, meta);
  return cudaGetLastError();
}
cudaError_t launch_rb_unpack(int* orig, int first, int n, int ext0, int batch, const int32_t* meta,
                             int32_t* res_path, float* res_margin, long long* ext_gid, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  k_rb_unpack<<<(n + 255) / 256 < 148 ? (n + 255) / 256 : 148, 256, 0, s>>>(orig, first, n, ext0, batch, meta,
                                                                            res_path, res_margin, ext_gid);
  return cudaGetLastError();
}
cudaError_t launch_rb_return(const int* sent_orig, int n, int K, const float* ret_logits, const int32_t* ret_path,
                             const float* ret_margin, float* res_logits, int32_t* res_path, float* res_margin,
                             cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int blocks = (n + 7) / 8;
  if (blocks > 148 * 4) blocks = 148 * 4;
  k_rb_return<<<blocks, 256, 0, s>>>(sent_orig, n, K, ret_logits, ret_path, ret_margin, res_logits, res_path,
                                     res_margin);
  return cudaGetLastError();
}
cudaError_t launch_set_int(int* p, int v, cudaStream_t s) {
  k_set_int<<<1, 1, 0, s>>>(p, v);
  return cudaGetLastError();
}

bool& pdl_flag() {
  thread_local bool on = false;
  return on;
}

// Lazy-loading anchor: a kernel of this translation unit's module (preload_kernels, hostmod.cu).
__global__ void k_tu_anchor_hostmod() {}
const void* tu_anchor_hostmod() { return reinterpret_cast<const void*>(&k_tu_anchor_hostmod); }

}  // namespace dycl
