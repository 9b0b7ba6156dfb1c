// libdycl: the image-captioning En-Decoder's decoder.
//
// The generative DyNN of the paper's study whose encoder is a CNN: here the encoder is an image
// graph (dycl_graph, its final tensor exported through dycl_io.features) and this graph is the
// decoder loop under the loop guard -- the `If` on the output token (L265) and the constant
// iteration bound (L267-268).  Per step, over the still-active captions only (compacted by
// k_compact; the LSTM state and the annotation vectors stay in slot order):
//   k_cap_gather   word embedding E[y] and the bf16 copy of h into the gate GEMM's A row, h also
//                  into the query GEMM's operand
//   q GEMM         q = W_q h + b_q                         (k_gemm_tma, fp32 out)
//   k_cap_attend   alpha = softmax_j(a_j . q / sqrt(D)), z = sum_j alpha_j a_j -> the A row
//   gate GEMM      [E[y]; z; h] W^T + b                    (k_gemm_tma, fp32 out)
//   k_cap_lstm     c, h update of the row's slot; bf16 h for the output GEMM
//   output GEMM    logits = W_o h + b_o with the argmax in its epilogue (no logits in HBM)
//   k_argmax_final token, top-1 logit, done flag;  k_compact  the active set
// Numerics (oracle mirror mode, reading R20): bf16 tensor-core operands (E rows, z, h, mean(a)),
// fp32 state / q / attention weights / logits.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <new>
#include <string>
#include <vector>

#include "../../include/dycl.h"
#include "epilogue.cuh"
#include "kernels.h"
#include "s2s_kernels.h"

namespace dycl {
namespace {

__device__ __forceinline__ float bfv(uint16_t u) { return __uint_as_float((uint32_t)u << 16); }
__device__ __forceinline__ uint16_t to_bf16(float f) {
  __nv_bfloat16 h = __float2bfloat16_rn(f);
  return *reinterpret_cast<uint16_t*>(&h);
}
__device__ __forceinline__ float sigm(float x) { return 1.0f / (1.0f + expf(-x)); }

struct CapStepArgs {
  const int32_t* active;     // row -> slot
  const int* n_live;
  const uint16_t* feat;      // [B][L][D] bf16 annotation vectors (slot order)
  const uint16_t* emb;       // [V][E] bf16
  const int32_t* cur_tok;    // [B] token fed this step (slot)
  float* h32;                // [B][H] state (slot)
  float* c32;                // [B][H]
  uint16_t* A;               // [rows][E + D + H] gate GEMM operand (row order)
  uint16_t* hb;              // [rows][H] bf16 h (row order)
  const float* q;            // [rows][D]
  const float* gates;        // [rows][4H]
  int E, D, H, L;
};

// abar = mean_j a_j (fp32, fixed order j ascending) -> bf16 [B][D]; warp per caption, lane = 2 dims
__global__ void k_cap_mean(const uint16_t* __restrict__ feat, uint16_t* __restrict__ abar, int B, int L, int D) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= B) return;
  const uint16_t* f = feat + (size_t)row * L * D;
  for (int d = lane; d < D; d += 32) {
    float s = 0.f;
    for (int j = 0; j < L; ++j) s += bfv(f[(size_t)j * D + d]);
    abar[(size_t)row * D + d] = to_bf16(s / (float)L);
  }
}

// h0 = tanh(pre[:H]), c0 = tanh(pre[H:]) of slot = row (active = iota at t = 0)
__global__ void k_cap_init_state(const float* __restrict__ pre, float* h32, float* c32, int B, int H) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)B * H) return;
  const long long r = i / H;
  const int k = (int)(i - r * H);
  h32[i] = tanhf(pre[r * 2 * H + k]);
  c32[i] = tanhf(pre[r * 2 * H + H + k]);
}

// A[row] = [E[y] | (z later) | bf16(h)], hb[row] = bf16(h); thread per (row, 8-element chunk)
__global__ void k_cap_gather(const CapStepArgs a) {
  const int n = *a.n_live;
  const int K = a.E + a.D + a.H;
  const int ce = a.E / 8, ch = a.H / 8;
  const long long total = (long long)n * (ce + ch);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(i / (ce + ch)), u = (int)(i - (long long)row * (ce + ch));
    const int slot = a.active[row];
    if (u < ce) {
      const uint4 v = *reinterpret_cast<const uint4*>(a.emb + (size_t)a.cur_tok[slot] * a.E + u * 8);
      *reinterpret_cast<uint4*>(a.A + (size_t)row * K + u * 8) = v;
    } else {
      const int k = (u - ce) * 8;
      const float* hp = a.h32 + (size_t)slot * a.H + k;
      const float4 h0 = *reinterpret_cast<const float4*>(hp), h1 = *reinterpret_cast<const float4*>(hp + 4);
      const uint4 o = make_uint4(pack_bf16x2_rn(h0.x, h0.y), pack_bf16x2_rn(h0.z, h0.w), pack_bf16x2_rn(h1.x, h1.y),
                                 pack_bf16x2_rn(h1.z, h1.w));
      *reinterpret_cast<uint4*>(a.A + (size_t)row * K + a.E + a.D + k) = o;
      *reinterpret_cast<uint4*>(a.hb + (size_t)row * a.H + k) = o;
    }
  }
}

// soft attention, warp per active row (D = 64: lane owns dims 2 lane, 2 lane + 1; L <= 64:
// lane owns keys lane, lane + 32); fixed-order reductions
__global__ void k_cap_attend(const CapStepArgs a) {
  const int n = *a.n_live;
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= n) return;
  const int slot = a.active[row];
  const uint16_t* f = a.feat + (size_t)slot * a.L * a.D;
  const float* q = a.q + (size_t)row * a.D;
  const float q0 = q[2 * lane], q1 = q[2 * lane + 1];
  const float scale = rsqrtf((float)a.D);
  float e[2];
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    const int j = lane + 32 * hh;
    float s = 0.f;
    for (int d = 0; d < a.D; d += 2) {
      const float qa = __shfl_sync(0xffffffffu, q0, d >> 1), qb = __shfl_sync(0xffffffffu, q1, d >> 1);
      if (j < a.L) {
        const uint32_t w = *reinterpret_cast<const uint32_t*>(f + (size_t)j * a.D + d);
        s = fmaf(qa, __uint_as_float(w << 16), s);
        s = fmaf(qb, __uint_as_float(w & 0xFFFF0000u), s);
      }
    }
    e[hh] = j < a.L ? s * scale : -INFINITY;
  }
  float m = fmaxf(e[0], e[1]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  const float p0 = lane < a.L ? expf(e[0] - m) : 0.f, p1 = lane + 32 < a.L ? expf(e[1] - m) : 0.f;
  float sum = p0 + p1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float inv = 1.0f / sum;
  float z0 = 0.f, z1 = 0.f;
  for (int j = 0; j < a.L; ++j) {
    const float al = __shfl_sync(0xffffffffu, j < 32 ? p0 : p1, j & 31) * inv;
    const uint32_t w = *reinterpret_cast<const uint32_t*>(f + (size_t)j * a.D + 2 * lane);
    z0 = fmaf(al, __uint_as_float(w << 16), z0);
    z1 = fmaf(al, __uint_as_float(w & 0xFFFF0000u), z1);
  }
  const int K = a.E + a.D + a.H;
  *reinterpret_cast<uint32_t*>(a.A + (size_t)row * K + a.E + 2 * lane) = pack_bf16x2_rn(z0, z1);
}

// LSTM cell of the row's slot (gate order i, f, g, o); bf16 h for the output GEMM
__global__ void k_cap_lstm(const CapStepArgs a) {
  const int n = *a.n_live;
  const long long total = (long long)n * a.H;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(i / a.H), k = (int)(i - (long long)row * a.H);
    const int slot = a.active[row];
    const float* g = a.gates + (size_t)row * 4 * a.H;
    const float ig = sigm(g[k]), fg = sigm(g[a.H + k]), gg = tanhf(g[2 * a.H + k]), og = sigm(g[3 * a.H + k]);
    float* cp = a.c32 + (size_t)slot * a.H + k;
    const float c = fg * *cp + ig * gg;
    const float h = og * tanhf(c);
    *cp = c;
    a.h32[(size_t)slot * a.H + k] = h;
    a.hb[(size_t)row * a.H + k] = to_bf16(h);
  }
}

int blocks_for(long long work, int threads, int num_sms) {
  long long b = (work + threads - 1) / threads;
  if (b > (long long)num_sms * 16) b = (long long)num_sms * 16;
  return b < 1 ? 1 : (int)b;
}

}  // namespace
// Lazy-loading anchor: a kernel of this translation unit's module (preload_kernels, hostmod.cu).
__global__ void k_tu_anchor_cap() {}
const void* tu_anchor_cap() { return reinterpret_cast<const void*>(&k_tu_anchor_cap); }

}  // namespace dycl

struct dycl_cap_s {
  dycl_cap_config c{};
  int device = 0, num_sms = 148;
  std::string err;
  std::vector<void*> allocs;
  bool finalized = false;
  int64_t max_batch = 0;
  uint16_t *init_w = nullptr, *att_w = nullptr, *emb = nullptr, *lstm_w = nullptr, *out_w = nullptr;
  float *init_b = nullptr, *att_b = nullptr, *lstm_b = nullptr, *out_b = nullptr;
  // workspace
  uint16_t *abar = nullptr, *A = nullptr, *hb = nullptr;
  float *pre = nullptr, *h32 = nullptr, *c32 = nullptr, *q = nullptr, *gates = nullptr, *am_val = nullptr;
  int *am_idx = nullptr, *counts = nullptr;
  int32_t *cur_tok = nullptr, *active[2] = {}, *list1 = nullptr, *list0 = nullptr, *zero_i = nullptr;
  float* zero_f = nullptr;
  uint8_t* flag = nullptr;
  int launches = 0;
  // CUDA graph of a whole run (init + max_len guarded steps), captured on first use per
  // (io pointers, batch) and replayed: every kernel sizes itself from device counts
  bool use_graph = true;             // DYCL_CAP_GRAPH=0 disables
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t gexec = nullptr;
  const void* gkey[4] = {};
  int64_t gbatch = -1;
  int glaunches = 0;
};

static thread_local std::string g_cap_err;

namespace {

dycl_status cfail(dycl_cap c, dycl_status st, const std::string& m) {
  if (c) c->err = m; else g_cap_err = m;
  return st;
}
template <typename T>
dycl_status cup(dycl_cap c, T** dst, const T* src, size_t n) {
  if (!src) return cfail(c, DYCL_E_INVALID_ARG, "null weight pointer");
  void* p = nullptr;
  if (cudaMalloc(&p, n * sizeof(T)) != cudaSuccess) return cfail(c, DYCL_E_OOM, "cudaMalloc (weights)");
  c->allocs.push_back(p);
  if (cudaMemcpy(p, src, n * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess)
    return cfail(c, DYCL_E_CUDA, "weight upload");
  *dst = static_cast<T*>(p);
  return DYCL_OK;
}
template <typename T>
dycl_status calloc_(dycl_cap c, T** dst, size_t n) {
  void* p = nullptr;
  if (cudaMalloc(&p, (n ? n : 1) * sizeof(T)) != cudaSuccess) return cfail(c, DYCL_E_OOM, "cudaMalloc (workspace)");
  c->allocs.push_back(p);
  *dst = static_cast<T*>(p);
  return DYCL_OK;
}

// y = A W^T + b over rows [0, *cnt) (or n_static) on the tcgen05 dense GEMM, fp32 out
cudaError_t gemm32(dycl_cap c, const uint16_t* A, int K, const uint16_t* w, const float* b, int N, float* y,
                   const int* cnt, int n_static, int max_rows, cudaStream_t st, const dycl::ConvArgs* am = nullptr) {
  dycl::ConvArgs a{};
  if (am) a = *am;
  a.x = A; a.w = w; a.bias = b; a.y = nullptr; a.y32 = y; a.n_live = cnt; a.n_static = n_static;
  a.H = a.W = a.Ho = a.Wo = 1; a.C = K; a.Cout = N; a.ksz = 1; a.stride = 1; a.pad = 0; a.K = K; a.Kp = K;
  a.rH = a.rW = 1; a.rC = N; a.nhwc = a.in_nhwc = 0;
  ++c->launches;
  return dycl::launch_gemm_tma(a, max_rows, c->num_sms, st);
}

}  // namespace

extern "C" {

dycl_status dycl_cap_create(int cuda_device, const dycl_cap_config* cfg, dycl_cap* out) {
  if (!cfg || !out) return cfail(nullptr, DYCL_E_INVALID_ARG, "null argument");
  *out = nullptr;
  const int K = cfg->emb + cfg->feat_dim + cfg->hidden;
  if (cfg->feat_dim != 64 || cfg->feat_len < 1 || cfg->feat_len > 64 || cfg->hidden % 64 || cfg->emb % 64 ||
      K % 64 || cfg->vocab % 256 || cfg->max_len < 1 || cfg->max_len > 64 || cfg->eos < 0 || cfg->eos >= cfg->vocab ||
      cfg->bos < 0 || cfg->bos >= cfg->vocab)
    return cfail(nullptr, DYCL_E_UNSUPPORTED,
                 "caption config: feat_dim 64, feat_len <= 64, hidden / emb multiples of 64, vocab of 256, max_len <= 64");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return cfail(nullptr, DYCL_E_CUDA, "no CUDA device");
  if (cuda_device < 0 || cuda_device >= ndev) return cfail(nullptr, DYCL_E_INVALID_ARG, "bad device index");
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, cuda_device);
  if (major != 10) return cfail(nullptr, DYCL_E_UNSUPPORTED, "libdycl is built for sm_100a (B200) only");
  dycl_cap c = new (std::nothrow) dycl_cap_s();
  if (!c) return cfail(nullptr, DYCL_E_OOM, "host allocation");
  c->c = *cfg;
  c->device = cuda_device;
  if (const char* eg = getenv("DYCL_CAP_GRAPH")) c->use_graph = atoi(eg) != 0;
  cudaSetDevice(cuda_device);
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, cuda_device);
  *out = c;
  return DYCL_OK;
}

dycl_status dycl_cap_destroy(dycl_cap c) {
  if (!c) return DYCL_OK;
  cudaSetDevice(c->device);
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  for (void* p : c->allocs) cudaFree(p);
  delete c;
  return DYCL_OK;
}

const char* dycl_cap_last_error(dycl_cap c) { return c ? c->err.c_str() : g_cap_err.c_str(); }

dycl_status dycl_cap_set_weights(dycl_cap c, const uint16_t* init_w, const float* init_b, const uint16_t* att_w,
                                 const float* att_b, const uint16_t* emb, const uint16_t* lstm_w, const float* lstm_b,
                                 const uint16_t* out_w, const float* out_b) {
  if (!c) return DYCL_E_INVALID_ARG;
  if (c->finalized) return cfail(c, DYCL_E_STATE, "already finalized");
  if (c->init_w) return cfail(c, DYCL_E_STATE, "weights already set");
  cudaSetDevice(c->device);
  const size_t V = c->c.vocab, E = c->c.emb, H = c->c.hidden, D = c->c.feat_dim;
  dycl_status r;
  if ((r = cup(c, &c->init_w, init_w, 2 * H * D)) || (r = cup(c, &c->init_b, init_b, 2 * H)) ||
      (r = cup(c, &c->att_w, att_w, D * H)) || (r = cup(c, &c->att_b, att_b, D)) ||
      (r = cup(c, &c->emb, emb, V * E)) || (r = cup(c, &c->lstm_w, lstm_w, 4 * H * (E + D + H))) ||
      (r = cup(c, &c->lstm_b, lstm_b, 4 * H)) || (r = cup(c, &c->out_w, out_w, V * H)) ||
      (r = cup(c, &c->out_b, out_b, V)))
    return r;
  return DYCL_OK;
}

dycl_status dycl_cap_finalize(dycl_cap c, int64_t max_batch) {
  if (!c) return DYCL_E_INVALID_ARG;
  if (c->finalized) return cfail(c, DYCL_E_STATE, "already finalized");
  if (!c->init_w) return cfail(c, DYCL_E_STATE, "weights not set");
  if (max_batch < 1 || max_batch > (1 << 20)) return cfail(c, DYCL_E_INVALID_ARG, "bad max_batch");
  cudaSetDevice(c->device);
  const size_t B = max_batch, V = c->c.vocab, E = c->c.emb, H = c->c.hidden, D = c->c.feat_dim;
  dycl_status r;
  if ((r = calloc_(c, &c->abar, B * D)) || (r = calloc_(c, &c->A, B * (E + D + H))) || (r = calloc_(c, &c->hb, B * H)) ||
      (r = calloc_(c, &c->pre, B * 2 * H)) || (r = calloc_(c, &c->h32, B * H)) || (r = calloc_(c, &c->c32, B * H)) ||
      (r = calloc_(c, &c->q, B * D)) || (r = calloc_(c, &c->gates, B * 4 * H)) ||
      (r = calloc_(c, &c->am_val, B * (V / 64))) || (r = calloc_(c, &c->am_idx, B * (V / 64))) ||
      (r = calloc_(c, &c->counts, 2 + 2 * (size_t)c->c.max_len)) || (r = calloc_(c, &c->cur_tok, B)) ||
      (r = calloc_(c, &c->active[0], B)) || (r = calloc_(c, &c->active[1], B)) || (r = calloc_(c, &c->list1, B)) ||
      (r = calloc_(c, &c->list0, B)) || (r = calloc_(c, &c->flag, B)) || (r = calloc_(c, &c->zero_i, 1)) ||
      (r = calloc_(c, &c->zero_f, 1)))
    return r;
  if (cudaMemset(c->zero_i, 0, 4) != cudaSuccess || cudaMemset(c->zero_f, 0, 4) != cudaSuccess)
    return cfail(c, DYCL_E_CUDA, "memset");
  c->max_batch = max_batch;
  c->finalized = true;
  return DYCL_OK;
}

}  // extern "C"

static dycl_status cap_enqueue(dycl_cap c, const uint16_t* features, int64_t batch, int32_t* tokens, int32_t* lengths,
                               float* top1, cudaStream_t st) {
  const dycl_cap_config& k = c->c;
  const int B = (int)batch, E = k.emb, H = k.hidden, D = k.feat_dim, L = k.feat_len, V = k.vocab;
  const int K = E + D + H;
  c->launches = 0;
  cudaError_t e;
#define CE(x)                                                                                          \
  do {                                                                                                 \
    e = (x);                                                                                           \
    if (e != cudaSuccess) return cfail(c, DYCL_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e)); \
  } while (0)
  dycl::S2SInitArgs ia{tokens, top1, c->cur_tok, lengths, c->active[0], c->counts, B, k.max_len, k.pad, k.bos};
  CE(dycl::launch_s2s_init(ia, st));
  // h0, c0 from the mean annotation vector
  dycl::k_cap_mean<<<dycl::blocks_for((long long)B * 32, 256, 1 << 20), 256, 0, st>>>(features, c->abar, B, L, D);
  CE(cudaGetLastError());
  CE(gemm32(c, c->abar, D, c->init_w, c->init_b, 2 * H, c->pre, nullptr, B, B, st));
  dycl::k_cap_init_state<<<dycl::blocks_for((long long)B * H, 256, 1 << 20), 256, 0, st>>>(c->pre, c->h32, c->c32, B, H);
  CE(cudaGetLastError());
  c->launches += 3;
  int cur = 0;
  const int* cnt = c->counts;
  for (int t = 0; t < k.max_len; ++t) {
    dycl::CapStepArgs sa{};
    sa.active = c->active[cur]; sa.n_live = cnt; sa.feat = features; sa.emb = c->emb; sa.cur_tok = c->cur_tok;
    sa.h32 = c->h32; sa.c32 = c->c32; sa.A = c->A; sa.hb = c->hb; sa.q = c->q; sa.gates = c->gates;
    sa.E = E; sa.D = D; sa.H = H; sa.L = L;
    dycl::k_cap_gather<<<dycl::blocks_for((long long)B * (E + H) / 8, 256, c->num_sms), 256, 0, st>>>(sa);
    CE(cudaGetLastError());
    CE(gemm32(c, c->hb, H, c->att_w, c->att_b, D, c->q, cnt, 0, B, st));
    dycl::k_cap_attend<<<dycl::blocks_for((long long)B * 32, 256, 1 << 20), 256, 0, st>>>(sa);
    CE(cudaGetLastError());
    CE(gemm32(c, c->A, K, c->lstm_w, c->lstm_b, 4 * H, c->gates, cnt, 0, B, st));
    dycl::k_cap_lstm<<<dycl::blocks_for((long long)B * H, 256, c->num_sms), 256, 0, st>>>(sa);
    CE(cudaGetLastError());
    // logits with the argmax in the GEMM epilogue (plain guard: no length bias)
    dycl::ConvArgs am{};
    am.am_val = c->am_val; am.am_idx = c->am_idx;
    am.g_slot = c->active[cur]; am.g_src = c->zero_i; am.g_len = c->zero_f; am.g_beta = 0.f;
    am.g_t = t; am.g_S = 0; am.g_eos = k.eos;
    CE(gemm32(c, c->hb, H, c->out_w, c->out_b, V, nullptr, cnt, 0, B, st, &am));
    dycl::S2SArgmaxArgs ga{nullptr, c->active[cur], c->zero_i, c->zero_f, 0.f, tokens, top1, nullptr,
                           c->cur_tok, lengths, c->flag, cnt, V, 0, k.max_len, t, k.eos};
    ga.am_val = c->am_val; ga.am_idx = c->am_idx;
    dycl::ConvArgs probe{};
    probe.Cout = V;
    ga.ntiles = V / dycl::gemm_tma_bn(probe, B, c->num_sms);
    CE(dycl::launch_argmax_final(ga, B, st));
    int* out_counts = c->counts + 1 + 2 * t;
    CE(dycl::launch_compact(c->flag, cnt, c->active[cur], c->list1, c->list0, out_counts, c->active[cur ^ 1], 0,
                            nullptr, 0, nullptr, 0.f, nullptr, st));
    c->launches += 5;
    cnt = out_counts + 1;
    cur ^= 1;
  }
#undef CE
  return DYCL_OK;
}

extern "C" {

dycl_status dycl_cap_run(dycl_cap c, const uint16_t* features, int64_t batch, int32_t* tokens, int32_t* lengths,
                         float* top1, void* stream) {
  if (!c) return DYCL_E_INVALID_ARG;
  if (!c->finalized) return cfail(c, DYCL_E_STATE, "not finalized");
  if (batch < 0 || batch > c->max_batch) return cfail(c, DYCL_E_SHAPE_MISMATCH, "batch > max_batch");
  if (batch == 0) return DYCL_OK;
  if (!features || !tokens || !lengths) return cfail(c, DYCL_E_INVALID_ARG, "null io pointer");
  if (cudaSetDevice(c->device) != cudaSuccess) return cfail(c, DYCL_E_CUDA, "cudaSetDevice");
  if (cudaError_t e = cudaGetLastError()) return cfail(c, DYCL_E_CUDA, cudaGetErrorString(e));
  cudaStream_t st = (cudaStream_t)stream;
  if (!c->use_graph) return cap_enqueue(c, features, batch, tokens, lengths, top1, st);
  const void* key[4] = {features, tokens, lengths, top1};
  bool hit = c->gexec && c->gbatch == batch;
  for (int i = 0; i < 4 && hit; ++i) hit = key[i] == c->gkey[i];
  if (!hit) {
    if (c->gexec) {
      cudaGraphExecDestroy(c->gexec);
      c->gexec = nullptr;
    }
    if (!c->cap_stream && cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking) != cudaSuccess)
      return cfail(c, DYCL_E_CUDA, "stream create");
    if (cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
      return cfail(c, DYCL_E_CUDA, "begin capture");
    dycl_status r = cap_enqueue(c, features, batch, tokens, lengths, top1, c->cap_stream);
    cudaGraph_t graph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(c->cap_stream, &graph);
    if (r != DYCL_OK) {
      if (graph) cudaGraphDestroy(graph);
      return r;
    }
    if (ec != cudaSuccess) return cfail(c, DYCL_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(ec));
    const cudaError_t ei = cudaGraphInstantiate(&c->gexec, graph, 0);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) {
      c->gexec = nullptr;
      return cfail(c, DYCL_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ei));
    }
    for (int i = 0; i < 4; ++i) c->gkey[i] = key[i];
    c->gbatch = batch;
    c->glaunches = c->launches;
  }
  if (cudaError_t e = cudaGraphLaunch(c->gexec, st)) return cfail(c, DYCL_E_CUDA, cudaGetErrorString(e));
  c->launches = c->glaunches;
  return DYCL_OK;
}

dycl_status dycl_cap_launches(dycl_cap c, int32_t* out) {
  if (!c || !out) return DYCL_E_INVALID_ARG;
  *out = c->launches;
  return DYCL_OK;
}

}  // extern "C"
