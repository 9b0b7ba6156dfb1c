// libdycl: the generative-DyNN graph (config 4) -- registration, loop-guard executor.
//
// P_Host for a generative DyNN: run the encoder sub-network
// once, then the decoder-step sub-network inside a loop bounded by the constant max_len;
// the logic node on the output token (EOS / length guard) runs on the device every step
// and the still-active sequences are compacted (k_compact), so the next step's kernels
// process exactly the active rows.  KV caches stay in slot order (rows carry their slot).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/dycl.h"
#include "kernels.h"
#include "s2s_kernels.h"

namespace {

struct DevLayer {
  uint16_t *wqkv = nullptr, *wo = nullptr, *wq2 = nullptr, *wkv2 = nullptr, *wo2 = nullptr, *w1 = nullptr,
           *w2 = nullptr;
  float *bqkv = nullptr, *bo = nullptr, *bq2 = nullptr, *bkv2 = nullptr, *bo2 = nullptr, *b1 = nullptr, *b2 = nullptr;
  float *lsg = nullptr, *lsb = nullptr, *lcg = nullptr, *lcb = nullptr, *lfg = nullptr, *lfb = nullptr;
};

}  // namespace

struct dycl_s2s_s {
  dycl_s2s_config c{};
  int device = 0, num_sms = 148;
  std::string err;
  std::vector<void*> allocs;
  std::vector<DevLayer> enc, dec;
  uint16_t *src_emb = nullptr, *tgt_emb = nullptr, *lm_w = nullptr;
  float *lm_b = nullptr, *len_table = nullptr;
  float beta = 0.f;
  bool finalized = false;
  int64_t max_batch = 0;
  // workspace
  float *x32 = nullptr, *pre = nullptr, *logits = nullptr;
  uint16_t *xb = nullptr, *qkv = nullptr, *att = nullptr, *h = nullptr;
  std::vector<uint16_t*> cross, cache;
  int32_t *cur_tok = nullptr, *active[2] = {}, *list1 = nullptr, *list0 = nullptr;
  int* counts = nullptr;
  uint8_t* flag = nullptr;
  int32_t *src_stage = nullptr, *tok_stage = nullptr, *len_stage = nullptr;
  int launches = 0;
  // CUDA graph of one whole run (encoder + the max_len guarded decode steps, ~4.5k kernels):
  // captured on first use for an (io pointers, batch) key, replayed on the caller's stream.
  // Every kernel reads its live row count from device memory, so the captured sequence is
  // valid for any data; only the pointers and the batch are baked in.
  bool use_graph = true;             // DYCL_S2S_GRAPH=0 disables
  bool pdl = true;                   // programmatic dependent launch in the run (DYCL_S2S_PDL=0 disables)
  int gemm_path = 0;                 // 0: k_gemm_tma, 1: k_conv_gemm (DYCL_S2S_GEMM=1; measured equal or slower)
  bool fuse_argmax = true;           // LM-head argmax in the GEMM epilogue (DYCL_S2S_FUSE_ARGMAX=0 disables)
  float* am_val = nullptr;           // fused argmax partials [max_batch][vocab / 64]
  int* am_idx = nullptr;
  // residual + LayerNorm in the epilogue of the out-proj / FFN-down GEMMs (decode steps and the
  // encoder; ConvArgs.ln_*; DYCL_S2S_FUSE_LN=0 disables): row partials and per-M-tile counters
  bool fuse_ln = true;
  float* ln_part = nullptr;          // [max_batch * src_len][d / 64] (sum, M2) pairs
  int* ln_cnt = nullptr;             // one per 128-row M tile, zero between launches
  // DYCL_PREC_BF16X3_PARITY: every bf16 tensor is a split pair [hi | lo] and every GEMM runs
  // on K-concatenated operands [A_hi | A_lo] x [W | W] (weights are exact bf16, so the
  // W_lo terms of the 3-pass product vanish): fp32-accurate products on the tensor cores
  int pair = 0;
  // per-launch profiling (graph off while enabled)
  struct Rec {
    int kind;
    cudaEvent_t e0, e1;
    const int* cnt;                  // device live-row count, or nullptr -> rows
    int rows;
    double bpr, fpr, bfix;           // algorithmic bytes / flops per row, fixed bytes
  };
  bool profiling = false;
  std::vector<Rec> prof;
  size_t prof_used = 0;
  cudaStream_t prof_stream = nullptr;
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t gexec = nullptr;
  const void* gkey[6] = {};
  int64_t gbatch = -1;
  int glaunches = 0;
};

static thread_local std::string g_s2s_err;

namespace {

dycl_status sfail(dycl_s2s s, dycl_status st, const std::string& m) {
  if (s) s->err = m; else g_s2s_err = m;
  return st;
}
#define SCK(call)                                                                   \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) return sfail(s, DYCL_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

template <typename T>
dycl_status upload(dycl_s2s s, T** dst, const T* src, size_t n) {
  if (!src) return sfail(s, DYCL_E_INVALID_ARG, "null weight pointer");
  void* p = nullptr;
  if (cudaMalloc(&p, n * sizeof(T)) != cudaSuccess) return sfail(s, DYCL_E_OOM, "cudaMalloc (weights)");
  s->allocs.push_back(p);
  SCK(cudaMemcpy(p, src, n * sizeof(T), cudaMemcpyHostToDevice));
  *dst = static_cast<T*>(p);
  return DYCL_OK;
}
template <typename T>
dycl_status alloc(dycl_s2s s, T** dst, size_t n) {
  void* p = nullptr;
  if (cudaMalloc(&p, (n ? n : 1) * sizeof(T)) != cudaSuccess) return sfail(s, DYCL_E_OOM, "cudaMalloc (workspace)");
  s->allocs.push_back(p);
  *dst = static_cast<T*>(p);
  return DYCL_OK;
}

dycl_status add_layer(dycl_s2s s, const dycl_s2s_layer* w, bool decoder) {
  if (!s || !w) return DYCL_E_INVALID_ARG;
  if (s->finalized) return sfail(s, DYCL_E_STATE, "already finalized");
  const size_t d = s->c.d_model, f = s->c.d_ff;
  DevLayer L;
  dycl_status r;
  if ((r = upload(s, &L.wqkv, w->wqkv, 3 * d * d)) || (r = upload(s, &L.bqkv, w->bqkv, 3 * d)) ||
      (r = upload(s, &L.wo, w->wo, d * d)) || (r = upload(s, &L.bo, w->bo, d)) ||
      (r = upload(s, &L.lsg, w->ln_sa_g, d)) || (r = upload(s, &L.lsb, w->ln_sa_b, d)) ||
      (r = upload(s, &L.w1, w->w1, f * d)) || (r = upload(s, &L.b1, w->b1, f)) ||
      (r = upload(s, &L.w2, w->w2, d * f)) || (r = upload(s, &L.b2, w->b2, d)) ||
      (r = upload(s, &L.lfg, w->ln_ff_g, d)) || (r = upload(s, &L.lfb, w->ln_ff_b, d)))
    return r;
  if (decoder) {
    if ((r = upload(s, &L.wq2, w->wq2, d * d)) || (r = upload(s, &L.bq2, w->bq2, d)) ||
        (r = upload(s, &L.wkv2, w->wkv2, 2 * d * d)) || (r = upload(s, &L.bkv2, w->bkv2, 2 * d)) ||
        (r = upload(s, &L.wo2, w->wo2, d * d)) || (r = upload(s, &L.bo2, w->bo2, d)) ||
        (r = upload(s, &L.lcg, w->ln_ca_g, d)) || (r = upload(s, &L.lcb, w->ln_ca_b, d)))
      return r;
    s->dec.push_back(L);
  } else {
    s->enc.push_back(L);
  }
  return DYCL_OK;
}

struct S2SExec {
  dycl_s2s s;
  cudaStream_t st;
  int B;
  int n = 0;

  void pb(int kind, const int* cnt, int rows, double bpr, double fpr, double bfix) {
    if (!s->profiling) return;
    if (s->prof_used >= s->prof.size()) {
      dycl_s2s_s::Rec r{};
      cudaEventCreate(&r.e0);
      cudaEventCreate(&r.e1);
      s->prof.push_back(r);
    }
    dycl_s2s_s::Rec& r = s->prof[s->prof_used];
    r.kind = kind; r.cnt = cnt; r.rows = rows; r.bpr = bpr; r.fpr = fpr; r.bfix = bfix;
    cudaEventRecord(r.e0, st);
  }
  void pe() {
    if (!s->profiling) return;
    cudaEventRecord(s->prof[s->prof_used].e1, st);
    ++s->prof_used;
  }

  // y = act(x W^T + b [+ res]) on rows [0, *cnt) through the tcgen05 GEMM path (a dense
  // layer = 1x1 conv on [rows][1][1][K]).
  cudaError_t gemm(const uint16_t* x, int K, const uint16_t* w, const float* b, int N, const float* res32,
                   uint16_t* yb, float* y32, int relu, const int* cnt, int n_static, int max_rows,
                   const dycl::ConvArgs* argmax = nullptr) {
    dycl::ConvArgs a{};
    if (argmax) a = *argmax;           // the fused-argmax fields (LM head)
    if (s->pair) {                     // [A_hi | A_lo] x [W | W], bf16 outputs written as pairs
      K *= 2;
      a.split = yb != nullptr;
    }
    a.x = x; a.w = w; a.bias = b; a.res32 = res32; a.res_mode = res32 ? 1 : 0;
    a.y = yb; a.y32 = y32; a.n_live = cnt; a.n_static = n_static;
    a.H = a.W = a.Ho = a.Wo = 1; a.C = K; a.Cout = N; a.ksz = 1; a.stride = 1; a.pad = 0;
    a.K = K; a.Kp = K; a.relu = relu;
    a.rH = a.rW = 1; a.rC = N;
    a.nhwc = a.in_nhwc = s->gemm_path;             // [rows][K] is NHWC at 1x1: the im2col-GEMM kernel
    ++n;
    pb(DYCL_K_GEMM, cnt, n_static, 2.0 * K + (yb ? 2.0 * N : 0.0) + (y32 ? 4.0 * N : 0.0) + (res32 ? 4.0 * N : 0.0) +
       (argmax ? 8.0 * N / dycl::gemm_tma_bn(a, max_rows, s->num_sms) : 0.0), 2.0 * K * N, 2.0 * K * N);
    const cudaError_t e = argmax ? dycl::launch_gemm_tma(a, max_rows, s->num_sms, st)
                                 : dycl::launch_conv(a, max_rows, s->num_sms, st, 0);
    pe();
    return e;
  }
  // x32 <- LN(x32 + x W^T + b), xb <- bf16 of it: one GEMM with the LayerNorm in its epilogue
  // when it applies, else the GEMM into `pre` followed by k_layernorm
  cudaError_t gemm_res_ln(const uint16_t* x, int K, const uint16_t* w, const float* b, const float* g,
                          const float* be, const int* cnt, int n_static, int max_rows) {
    const int d = s->c.d_model;
    dycl::ConvArgs a{};
    a.x = x; a.w = w; a.bias = b; a.res32 = s->x32; a.res_mode = 1;
    a.y = s->xb; a.y32 = s->x32; a.n_live = cnt; a.n_static = n_static;
    a.H = a.W = a.Ho = a.Wo = 1; a.C = K; a.Cout = d; a.ksz = 1; a.stride = 1; a.pad = 0;
    a.K = K; a.Kp = K; a.relu = 0;
    a.rH = a.rW = 1; a.rC = d;
    a.nhwc = a.in_nhwc = 1;
    if (!s->fuse_ln || s->pair || s->gemm_path || !dycl::gemm_tma_ln_ok(a, max_rows, s->num_sms)) {
      cudaError_t e = gemm(x, K, w, b, d, s->x32, nullptr, s->pre, 0, cnt, n_static, max_rows);
      return e != cudaSuccess ? e : ln(s->pre, g, be, cnt, n_static, max_rows);
    }
    a.ln_gamma = g; a.ln_beta = be; a.ln_part = s->ln_part; a.ln_cnt = s->ln_cnt; a.ln_eps = 1e-5f;
    ++n;
    pb(DYCL_K_GEMM, cnt, n_static, 2.0 * K + 2.0 * d + 4.0 * d + 4.0 * d, 2.0 * K * d + 8.0 * d, 2.0 * K * d);
    const cudaError_t e = dycl::launch_gemm_tma(a, max_rows, s->num_sms, st);
    pe();
    return e;
  }
  cudaError_t ln(const float* in, const float* g, const float* b, const int* cnt, int n_static, int max_rows) {
    dycl::S2SLnArgs a{in, g, b, s->x32, s->xb, cnt, n_static, s->c.d_model, 1e-5f};
    a.pair = s->pair;
    ++n;
    const double d = s->c.d_model;
    pb(DYCL_K_LN, cnt, n_static, 4.0 * d + 6.0 * d, 8.0 * d, 8.0 * d);
    const cudaError_t e = dycl::launch_layernorm(a, max_rows, st);
    pe();
    return e;
  }

  dycl_status run(const int32_t* src, int32_t* tokens, int32_t* lengths, float* top1, float* logits0) {
    const dycl_s2s_config& c = s->c;
    const int d = c.d_model, S = c.src_len, R = B * S;
    // the decode loop is ~70 dependent launches per step: each kernel's launch and prologue
    // overlap its predecessor's tail (per-launch profiling events would break the chain)
    dycl::PdlScope pdl_scope(s->pdl && !s->profiling);
    cudaError_t e;
#define E(x)                                                                        \
  do {                                                                              \
    e = (x);                                                                        \
    if (e != cudaSuccess) return sfail(s, DYCL_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e)); \
  } while (0)
    dycl::S2SInitArgs ia{tokens, top1, s->cur_tok, lengths, s->active[0], s->counts, B, c.max_len, c.pad, c.bos};
    pb(DYCL_K_INIT, nullptr, B, 4.0 * (c.max_len + 3), 0, 0);
    E(dycl::launch_s2s_init(ia, st));
    pe();
    ++n;
    // ---------------- encoder sub-network (once), rows = B*S tokens
    dycl::S2SEmbedArgs ea{s->src_emb, src, nullptr, nullptr, s->x32, s->xb, nullptr, R, d, S, 0};
    ea.pair = s->pair;
    pb(DYCL_K_EMBED, nullptr, R, 4.0 + 2.0 * d + 6.0 * d, 0, 0);
    E(dycl::launch_embed(ea, R, st));
    pe();
    ++n;
    for (const DevLayer& L : s->enc) {
      E(gemm(s->xb, d, L.wqkv, L.bqkv, 3 * d, nullptr, s->qkv, nullptr, 0, nullptr, R, R));
      dycl::S2SAttnArgs aa{};
      aa.qkv = s->qkv; aa.out = s->att; aa.n_static = B; aa.d = d; aa.heads = c.heads; aa.S = S;
      aa.pair = s->pair;
      pb(DYCL_K_ATTN, nullptr, B, (double)S * (3.0 * d * 2 + 2.0 * d), 4.0 * S * S * d, 0);
      E(dycl::launch_attn_encoder(aa, B, st));
      pe();
      ++n;
      // (the encoder keeps 256-wide N tiles + k_layernorm: its LN fused into 64-wide N tiles
      // measured 0.3 ms slower per batch -- at M = B*S the GEMM's tile width matters more)
      E(gemm(s->att, d, L.wo, L.bo, d, s->x32, nullptr, s->pre, 0, nullptr, R, R));
      E(ln(s->pre, L.lsg, L.lsb, nullptr, R, R));
      E(gemm(s->xb, d, L.w1, L.b1, c.d_ff, nullptr, s->h, nullptr, 1, nullptr, R, R));
      E(gemm(s->h, c.d_ff, L.w2, L.b2, d, s->x32, nullptr, s->pre, 0, nullptr, R, R));
      E(ln(s->pre, L.lfg, L.lfb, nullptr, R, R));
    }
    // cross-attention K/V of every decoder layer from the encoder output (bf16 operand copy)
    for (size_t l = 0; l < s->dec.size(); ++l)
      E(gemm(s->xb, d, s->dec[l].wkv2, s->dec[l].bkv2, 2 * d, nullptr, s->cross[l], nullptr, 0, nullptr, R, R));
    // ---------------- guarded greedy loop: t < max_len (the constant bound), active rows only
    int cur = 0;
    const int* cnt = s->counts;
    for (int t = 0; t < c.max_len; ++t) {
      const int32_t* slot = s->active[cur];
      dycl::S2SEmbedArgs de{s->tgt_emb, nullptr, slot, s->cur_tok, s->x32, s->xb, cnt, 0, d, S, t};
      de.pair = s->pair;
      pb(DYCL_K_EMBED, cnt, 0, 8.0 + 2.0 * d + 6.0 * d, 0, 0);
      E(dycl::launch_embed(de, B, st));
      pe();
      ++n;
      for (size_t l = 0; l < s->dec.size(); ++l) {
        const DevLayer& L = s->dec[l];
        E(gemm(s->xb, d, L.wqkv, L.bqkv, 3 * d, nullptr, s->qkv, nullptr, 0, cnt, 0, B));
        dycl::S2SAttnArgs sa{};
        sa.qkv = s->qkv; sa.q = s->qkv; sa.q_stride = (s->pair ? 6 : 3) * d; sa.kv = nullptr; sa.cache = s->cache[l];
        sa.pair = s->pair; sa.q_lo = 3 * d;
        sa.out = s->att; sa.slot = slot; sa.n_live = cnt; sa.d = d; sa.heads = c.heads; sa.S = S;
        sa.max_len = c.max_len; sa.t = t;
        pb(DYCL_K_ATTN, cnt, 0, (t + 1.0) * 2 * d * 2 + 3.0 * d * 2 + 2.0 * d * 2 + 2.0 * d * 2, 4.0 * (t + 1) * d, 0);
        E(dycl::launch_attn_decoder(sa, B, st));
        pe();
        ++n;
        E(gemm_res_ln(s->att, d, L.wo, L.bo, L.lsg, L.lsb, cnt, 0, B));
        E(gemm(s->xb, d, L.wq2, L.bq2, d, nullptr, s->att, nullptr, 0, cnt, 0, B));
        dycl::S2SAttnArgs ca{};
        ca.q = s->att; ca.q_stride = (s->pair ? 2 : 1) * d; ca.kv = s->cross[l]; ca.out = s->qkv;  // reuse qkv as scratch
        ca.pair = s->pair; ca.q_lo = d;
        ca.slot = slot; ca.n_live = cnt; ca.d = d; ca.heads = c.heads; ca.S = S; ca.max_len = c.max_len; ca.t = t;
        pb(DYCL_K_ATTN, cnt, 0, (double)S * 2 * d * 2 + 2.0 * d * 2 + 2.0 * d * 2, 4.0 * S * d, 0);
        E(dycl::launch_attn_decoder(ca, B, st));
        pe();
        ++n;
        E(gemm_res_ln(s->qkv, d, L.wo2, L.bo2, L.lcg, L.lcb, cnt, 0, B));
        E(gemm(s->xb, d, L.w1, L.b1, c.d_ff, nullptr, s->h, nullptr, 1, cnt, 0, B));
        E(gemm_res_ln(s->h, c.d_ff, L.w2, L.b2, L.lfg, L.lfb, cnt, 0, B));
      }
      dycl::S2SArgmaxArgs ga{s->logits, slot, src, s->len_table, s->beta, tokens, top1, logits0,
                             s->cur_tok, lengths, s->flag, cnt, c.vocab, S, c.max_len, t, c.eos};
      if (s->fuse_argmax && !(logits0 && t == 0)) {
        // LM head with the guard + argmax in its epilogue: per (row, N tile) the max and its
        // lowest index; the [rows][V] fp32 logits never reach HBM
        dycl::ConvArgs am{};
        am.am_val = s->am_val; am.am_idx = s->am_idx;
        am.g_slot = slot; am.g_src = src; am.g_len = s->len_table; am.g_beta = s->beta;
        am.g_t = t; am.g_S = S; am.g_eos = c.eos;
        E(gemm(s->xb, d, s->lm_w, s->lm_b, c.vocab, nullptr, nullptr, nullptr, 0, cnt, 0, B, &am));
        dycl::ConvArgs probe{};
        probe.Cout = c.vocab;
        ga.am_val = s->am_val; ga.am_idx = s->am_idx;
        ga.ntiles = c.vocab / dycl::gemm_tma_bn(probe, B, s->num_sms);
        pb(DYCL_K_ARGMAX, cnt, 0, 8.0 * ga.ntiles + 16.0, 0, 0);
        E(dycl::launch_argmax_final(ga, B, st));
      } else {
        E(gemm(s->xb, d, s->lm_w, s->lm_b, c.vocab, nullptr, nullptr, s->logits, 0, cnt, 0, B));
        pb(DYCL_K_ARGMAX, cnt, 0, 4.0 * c.vocab + 16.0, 2.0 * c.vocab, 0);
        E(dycl::launch_argmax_guard(ga, B, st));
      }
      pe();
      ++n;
      // the logic node's decision -> stable compaction of the still-active sequences
      int* out_counts = s->counts + 1 + 2 * t;
      pb(DYCL_K_COMPACT, cnt, 0, 1.0 + 12.0, 0, 0);
      E(dycl::launch_compact(s->flag, cnt, slot, s->list1, s->list0, out_counts, s->active[cur ^ 1], 0,
                             nullptr, 0, nullptr, 0.f, nullptr, st));
      pe();
      ++n;
      cnt = out_counts + 1;
      cur ^= 1;
    }
#undef E
    return DYCL_OK;
  }
};

}  // namespace

extern "C" {

dycl_status dycl_s2s_create(int cuda_device, const dycl_s2s_config* cfg, dycl_s2s* out) {
  if (!cfg || !out) return sfail(nullptr, DYCL_E_INVALID_ARG, "null argument");
  *out = nullptr;
  if (cfg->d_model % 64 || cfg->heads * 64 != cfg->d_model || cfg->d_model > 1024 || cfg->src_len < 1 ||
      cfg->src_len > 64 || cfg->max_len < 1 || cfg->max_len > 64 || cfg->vocab % 256 || cfg->d_ff % 256 ||
      cfg->enc_layers < 1 || cfg->dec_layers < 1 || cfg->eos < 0 || cfg->eos >= cfg->vocab)
    return sfail(nullptr, DYCL_E_UNSUPPORTED,
                 "s2s config: head dim 64, d_model <= 1024, src_len/max_len <= 64, vocab and d_ff multiples of 256");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return sfail(nullptr, DYCL_E_CUDA, "no CUDA device");
  if (cuda_device < 0 || cuda_device >= ndev) return sfail(nullptr, DYCL_E_INVALID_ARG, "bad device index");
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, cuda_device);
  if (major != 10) return sfail(nullptr, DYCL_E_UNSUPPORTED, "libdycl is built for sm_100a (B200) only");
  dycl_s2s s = new (std::nothrow) dycl_s2s_s();
  if (!s) return sfail(nullptr, DYCL_E_OOM, "host allocation");
  s->c = *cfg;
  s->device = cuda_device;
  if (const char* eg = getenv("DYCL_S2S_GRAPH")) s->use_graph = atoi(eg) != 0;
  if (const char* gp = getenv("DYCL_S2S_GEMM")) s->gemm_path = atoi(gp);
  if (const char* pp = getenv("DYCL_S2S_PDL")) s->pdl = atoi(pp) != 0;
  if (const char* fa = getenv("DYCL_S2S_FUSE_ARGMAX")) s->fuse_argmax = atoi(fa) != 0;
  if (const char* fl = getenv("DYCL_S2S_FUSE_LN")) s->fuse_ln = atoi(fl) != 0;
  cudaSetDevice(cuda_device);
  cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, cuda_device);
  *out = s;
  return DYCL_OK;
}

dycl_status dycl_s2s_destroy(dycl_s2s s) {
  if (!s) return DYCL_OK;
  cudaSetDevice(s->device);
  if (s->gexec) cudaGraphExecDestroy(s->gexec);
  for (auto& r : s->prof) {
    cudaEventDestroy(r.e0);
    cudaEventDestroy(r.e1);
  }
  if (s->cap_stream) cudaStreamDestroy(s->cap_stream);
  for (void* p : s->allocs) cudaFree(p);
  delete s;
  return DYCL_OK;
}

const char* dycl_s2s_last_error(dycl_s2s s) { return s ? s->err.c_str() : g_s2s_err.c_str(); }

dycl_status dycl_s2s_set_embeddings(dycl_s2s s, const uint16_t* src_emb, const uint16_t* tgt_emb) {
  if (!s) return DYCL_E_INVALID_ARG;
  if (s->finalized) return sfail(s, DYCL_E_STATE, "already finalized");
  cudaSetDevice(s->device);
  const size_t n = (size_t)s->c.vocab * s->c.d_model;
  if (dycl_status r = upload(s, &s->src_emb, src_emb, n)) return r;
  return upload(s, &s->tgt_emb, tgt_emb, n);
}

dycl_status dycl_s2s_add_encoder_layer(dycl_s2s s, const dycl_s2s_layer* w) {
  if (s) cudaSetDevice(s->device);
  return add_layer(s, w, false);
}
dycl_status dycl_s2s_add_decoder_layer(dycl_s2s s, const dycl_s2s_layer* w) {
  if (s) cudaSetDevice(s->device);
  return add_layer(s, w, true);
}

dycl_status dycl_s2s_set_lm_head(dycl_s2s s, const uint16_t* w, const float* b) {
  if (!s) return DYCL_E_INVALID_ARG;
  if (s->finalized) return sfail(s, DYCL_E_STATE, "already finalized");
  cudaSetDevice(s->device);
  if (dycl_status r = upload(s, &s->lm_w, w, (size_t)s->c.vocab * s->c.d_model)) return r;
  return upload(s, &s->lm_b, b, (size_t)s->c.vocab);
}

dycl_status dycl_s2s_set_loop_guard(dycl_s2s s, const float* len_table, float beta) {
  if (!s) return DYCL_E_INVALID_ARG;
  if (s->finalized) return sfail(s, DYCL_E_STATE, "already finalized");
  cudaSetDevice(s->device);
  s->beta = beta;
  std::vector<float> zeros;
  if (!len_table) {
    zeros.assign(s->c.vocab, 0.f);
    len_table = zeros.data();
  }
  return upload(s, &s->len_table, len_table, (size_t)s->c.vocab);
}

dycl_status dycl_s2s_set_precision(dycl_s2s s, int precision) {
  if (!s) return DYCL_E_INVALID_ARG;
  if (s->finalized) return sfail(s, DYCL_E_STATE, "already finalized");
  if (precision != DYCL_PREC_BF16 && precision != DYCL_PREC_BF16X3_PARITY)
    return sfail(s, DYCL_E_INVALID_ARG, "s2s precision: DYCL_PREC_BF16 or DYCL_PREC_BF16X3_PARITY");
  s->pair = precision == DYCL_PREC_BF16X3_PARITY;
  return DYCL_OK;
}

dycl_status dycl_s2s_finalize(dycl_s2s s, int64_t max_batch) {
  if (!s) return DYCL_E_INVALID_ARG;
  if (s->finalized) return sfail(s, DYCL_E_STATE, "already finalized");
  if (max_batch <= 0 || max_batch > 65536) return sfail(s, DYCL_E_INVALID_ARG, "bad max_batch");
  if (s->enc.size() != (size_t)s->c.enc_layers || s->dec.size() != (size_t)s->c.dec_layers || !s->src_emb ||
      !s->lm_w)
    return sfail(s, DYCL_E_STATE, "missing layers / embeddings / LM head");
  if (!s->len_table)
    if (dycl_status r = dycl_s2s_set_loop_guard(s, nullptr, 0.f)) return r;
  SCK(cudaSetDevice(s->device));
  const size_t B = max_batch, d = s->c.d_model, S = s->c.src_len, R = B * S, L = s->c.max_len;
  const size_t P = s->pair ? 2 : 1;               // split pairs double every bf16 tensor
  dycl_status r;
  if (s->pair) {                                  // [W | W] copies of every GEMM weight
    const size_t f = s->c.d_ff;
    auto dup = [&](uint16_t*& w, size_t N, size_t K) -> dycl_status {
      uint16_t* w2 = nullptr;
      if (dycl_status e = alloc(s, &w2, N * 2 * K)) return e;
      SCK(cudaMemcpy2D(w2, 4 * K, w, 2 * K, 2 * K, N, cudaMemcpyDeviceToDevice));
      SCK(cudaMemcpy2D(w2 + K, 4 * K, w, 2 * K, 2 * K, N, cudaMemcpyDeviceToDevice));
      w = w2;
      return DYCL_OK;
    };
    for (auto* Ls : {&s->enc, &s->dec})
      for (DevLayer& Lw : *Ls) {
        if ((r = dup(Lw.wqkv, 3 * d, d)) || (r = dup(Lw.wo, d, d)) || (r = dup(Lw.w1, f, d)) ||
            (r = dup(Lw.w2, d, f)))
          return r;
        if (Lw.wq2 && ((r = dup(Lw.wq2, d, d)) || (r = dup(Lw.wkv2, 2 * d, d)) || (r = dup(Lw.wo2, d, d))))
          return r;
      }
    if ((r = dup(s->lm_w, (size_t)s->c.vocab, d))) return r;
  }
  if ((r = alloc(s, &s->x32, R * d)) || (r = alloc(s, &s->pre, R * d)) || (r = alloc(s, &s->xb, R * d * P)) ||
      (r = alloc(s, &s->qkv, R * 3 * d * P)) || (r = alloc(s, &s->att, R * d * P)) ||
      (r = alloc(s, &s->h, R * (size_t)s->c.d_ff * P)) || (r = alloc(s, &s->logits, B * (size_t)s->c.vocab)) || (r = alloc(s, &s->am_val, B * (size_t)(s->c.vocab / 64))) ||
      (r = alloc(s, &s->am_idx, B * (size_t)(s->c.vocab / 64))) ||
      (r = alloc(s, &s->cur_tok, B)) || (r = alloc(s, &s->active[0], B)) || (r = alloc(s, &s->active[1], B)) ||
      (r = alloc(s, &s->list1, B)) || (r = alloc(s, &s->list0, B)) || (r = alloc(s, &s->counts, 2 * L + 2)) ||
      (r = alloc(s, &s->flag, B)) || (r = alloc(s, &s->ln_part, R * 2 * (size_t)(d / 64 + 1))) ||
      (r = alloc(s, &s->ln_cnt, R / 128 + 2)))
    return r;
  SCK(cudaMemset(s->ln_cnt, 0, (R / 128 + 2) * sizeof(int)));
  s->cross.resize(s->dec.size());
  s->cache.resize(s->dec.size());
  for (size_t l = 0; l < s->dec.size(); ++l)
    if ((r = alloc(s, &s->cross[l], R * 2 * d * P)) || (r = alloc(s, &s->cache[l], B * L * 2 * d * P))) return r;
  s->max_batch = max_batch;
  s->finalized = true;
  return DYCL_OK;
}

dycl_status dycl_s2s_run(dycl_s2s s, const int32_t* src, int64_t batch, int32_t* tokens, int32_t* lengths,
                         float* top1, float* logits0, void* stream) {
  if (!s) return DYCL_E_INVALID_ARG;
  if (!s->finalized) return sfail(s, DYCL_E_STATE, "not finalized");
  if (batch < 0 || batch > s->max_batch) return sfail(s, DYCL_E_SHAPE_MISMATCH, "batch > max_batch");
  if (batch == 0) return DYCL_OK;
  if (!src || !tokens || !lengths) return sfail(s, DYCL_E_INVALID_ARG, "null io pointer");
  SCK(cudaSetDevice(s->device));
  SCK(cudaGetLastError());
  if (!s->use_graph || s->profiling) {
    s->prof_used = 0;
    s->prof_stream = (cudaStream_t)stream;
    S2SExec ex{s, (cudaStream_t)stream, (int)batch};
    dycl_status r = ex.run(src, tokens, lengths, top1, logits0);
    s->launches = ex.n;
    return r;
  }
  const void* key[6] = {src, tokens, lengths, top1, logits0, nullptr};
  bool hit = s->gexec && s->gbatch == batch;
  for (int i = 0; i < 6 && hit; ++i) hit = key[i] == s->gkey[i];
  if (!hit) {
    if (s->gexec) {
      cudaGraphExecDestroy(s->gexec);
      s->gexec = nullptr;
    }
    if (!s->cap_stream) SCK(cudaStreamCreateWithFlags(&s->cap_stream, cudaStreamNonBlocking));
    SCK(cudaStreamBeginCapture(s->cap_stream, cudaStreamCaptureModeThreadLocal));
    S2SExec ex{s, s->cap_stream, (int)batch};
    dycl_status r = ex.run(src, tokens, lengths, top1, logits0);
    cudaGraph_t graph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(s->cap_stream, &graph);
    if (r != DYCL_OK) {
      if (graph) cudaGraphDestroy(graph);
      return r;
    }
    if (ec != cudaSuccess) return sfail(s, DYCL_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(ec));
    const cudaError_t ei = cudaGraphInstantiate(&s->gexec, graph, 0);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) {
      s->gexec = nullptr;
      return sfail(s, DYCL_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ei));
    }
    for (int i = 0; i < 6; ++i) s->gkey[i] = key[i];
    s->gbatch = batch;
    s->glaunches = ex.n;
  }
  SCK(cudaGraphLaunch(s->gexec, (cudaStream_t)stream));
  s->launches = s->glaunches;
  return DYCL_OK;
}

dycl_status dycl_s2s_run_host(dycl_s2s s, const int32_t* src_host, int64_t batch, int32_t* tokens_host,
                              int32_t* lengths_host, void* stream) {
  if (!s) return DYCL_E_INVALID_ARG;
  if (!s->finalized) return sfail(s, DYCL_E_STATE, "not finalized");
  if (batch < 0 || batch > s->max_batch) return sfail(s, DYCL_E_SHAPE_MISMATCH, "batch > max_batch");
  if (batch == 0) return DYCL_OK;
  SCK(cudaSetDevice(s->device));
  const size_t B = s->max_batch;
  if (!s->src_stage) {
    dycl_status r;
    if ((r = alloc(s, &s->src_stage, B * s->c.src_len)) || (r = alloc(s, &s->tok_stage, B * s->c.max_len)) ||
        (r = alloc(s, &s->len_stage, B)))
      return r;
  }
  cudaStream_t st = (cudaStream_t)stream;
  SCK(cudaMemcpyAsync(s->src_stage, src_host, (size_t)batch * s->c.src_len * 4, cudaMemcpyHostToDevice, st));
  if (dycl_status r = dycl_s2s_run(s, s->src_stage, batch, s->tok_stage, s->len_stage, nullptr, nullptr, stream))
    return r;
  SCK(cudaMemcpyAsync(tokens_host, s->tok_stage, (size_t)batch * s->c.max_len * 4, cudaMemcpyDeviceToHost, st));
  SCK(cudaMemcpyAsync(lengths_host, s->len_stage, (size_t)batch * 4, cudaMemcpyDeviceToHost, st));
  SCK(cudaStreamSynchronize(st));
  return DYCL_OK;
}

dycl_status dycl_s2s_set_profiling(dycl_s2s s, int enable) {
  if (!s) return DYCL_E_INVALID_ARG;
  s->profiling = enable != 0;
  return DYCL_OK;
}

dycl_status dycl_s2s_profile_read(dycl_s2s s, int32_t max_n, int32_t* kind, float* ms, double* bytes, double* flops,
                                  int32_t* n_out) {
  if (!s || !n_out) return DYCL_E_INVALID_ARG;
  SCK(cudaSetDevice(s->device));
  SCK(cudaStreamSynchronize(s->prof_stream));
  const int nslot = 1 + 2 * s->c.max_len;
  std::vector<int> counts(nslot, 0);
  if (s->counts) SCK(cudaMemcpy(counts.data(), s->counts, nslot * sizeof(int), cudaMemcpyDeviceToHost));
  const int n = (int)std::min<size_t>(s->prof_used, (size_t)std::max(max_n, 0));
  for (int i = 0; i < n; ++i) {
    const dycl_s2s_s::Rec& r = s->prof[i];
    float t = 0.f;
    SCK(cudaEventElapsedTime(&t, r.e0, r.e1));
    const double rows = r.cnt ? (double)counts[r.cnt - s->counts] : (double)r.rows;
    if (kind) kind[i] = r.kind;
    if (ms) ms[i] = t;
    if (bytes) bytes[i] = rows * r.bpr + r.bfix;
    if (flops) flops[i] = rows * r.fpr;
  }
  *n_out = (int32_t)s->prof_used;
  return DYCL_OK;
}

dycl_status dycl_s2s_launches(dycl_s2s s, int32_t* out) {
  if (!s || !out) return DYCL_E_INVALID_ARG;
  *out = s->launches;
  return DYCL_OK;
}

}  // extern "C"
