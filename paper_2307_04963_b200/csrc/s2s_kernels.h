// Config 4 kernel launchers (s2s_kernels.cu); internal to libdycl.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace dycl {

struct S2SEmbedArgs {
  const uint16_t* table;   // bf16 [V][d]
  const int32_t* src;      // encoder: tokens [B*S] (row = b*S + i), else nullptr
  const int32_t* slot;     // decoder: row -> sequence slot
  const int32_t* cur_tok;  // decoder: [B] token fed at step t
  float* x32;              // [rows][d]
  uint16_t* xb;            // [rows][d]
  const int* n_live;
  int n_static, d, S, t;
  int pair = 0;            // BF16X3 parity mode: xb rows are [hi(d) | lo(d)]
};
struct S2SLnArgs {
  const float* in;         // [rows][d]
  const float* gamma;
  const float* beta;
  float* out32;
  uint16_t* outb;
  const int* n_live;
  int n_static, d;
  float eps;
  int pair = 0;            // outb rows are [hi(d) | lo(d)]
};
struct S2SAttnArgs {
  const uint16_t* qkv;     // encoder: [B*S][3d]; decoder self: [rows][3d] (k, v appended)
  const uint16_t* q;       // decoder: query rows (stride q_stride)
  int q_stride;
  const uint16_t* kv;      // cross: [B][S][2d] encoder K/V; nullptr for self attention
  uint16_t* cache;         // self: [B][max_len][2d] this layer's K/V cache
  uint16_t* out;           // [rows][d]
  const int32_t* slot;
  const int* n_live;
  int n_static, d, heads, S, max_len, t;
  // BF16X3 parity mode: every bf16 tensor row is a split pair [hi | lo] (value = hi + lo):
  // qkv rows [q k v | q k v]_lo at +3d, K/V rows [K V | K V]_lo at +2d, out rows lo at +d;
  // q_lo = offset of the query's lo half within its row (3d self, d cross)
  int pair = 0;
  int q_lo = 0;
};
struct S2SArgmaxArgs {
  const float* logits;     // [rows][V]
  const int32_t* slot;
  const int32_t* src;      // [B][S]
  const float* len_table;  // [V]
  float beta;
  int32_t* tokens;         // [B][max_len]
  float* top1;             // [B][max_len] or nullptr
  float* logits0;          // [B][V] step-0 (biased) logits or nullptr
  int32_t* cur_tok;
  int32_t* lengths;
  uint8_t* flag;           // [rows] 1 = finished this step
  const int* n_live;
  int V, S, max_len, t, eos;
  // fused LM-head argmax: per-(row, N tile) partial maxima and their indices [rows][ntiles]
  const float* am_val = nullptr;
  const int* am_idx = nullptr;
  int ntiles = 0;
};
struct S2SInitArgs {
  int32_t* tokens;
  float* top1;
  int32_t* cur_tok;
  int32_t* lengths;
  int32_t* active;
  int* count;
  int B, max_len, pad, bos;
};

cudaError_t launch_embed(const S2SEmbedArgs& a, int max_rows, cudaStream_t s);
cudaError_t launch_layernorm(const S2SLnArgs& a, int max_rows, cudaStream_t s);
cudaError_t launch_attn_encoder(const S2SAttnArgs& a, int max_seqs, cudaStream_t s);
cudaError_t launch_attn_decoder(const S2SAttnArgs& a, int max_rows, cudaStream_t s);
cudaError_t launch_argmax_guard(const S2SArgmaxArgs& a, int max_rows, cudaStream_t s);
// the guard's decision from the fused LM-head partials (a.am_val / a.am_idx): one warp per row
cudaError_t launch_argmax_final(const S2SArgmaxArgs& a, int max_rows, cudaStream_t s);
cudaError_t launch_s2s_init(const S2SInitArgs& a, cudaStream_t s);

}  // namespace dycl
