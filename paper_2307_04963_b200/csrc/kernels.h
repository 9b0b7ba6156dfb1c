// Internal launcher interface between the runtime (api.cpp) and the sm_100a
// kernels.  Not part of the public ABI (that is include/dycl.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

namespace dycl {

// Implicit-GEMM convolution / dense layer on tcgen05 (conv_tc.cu).
//   rows  m = (sample n, ho, wo)  -> M = n_live * Ho * Wo
//   cols  o = output channel      -> N = Cout
//   depth k = (r, s, c)           -> K = ksz*ksz*C  (C % 8 == 0)
struct ConvArgs {
  const uint16_t* x;     // bf16 [n][H][W][C]
  const uint16_t* w;     // bf16 [Cout][Kp]  (K zero-padded to Kp = roundup(K, 64))
  const uint16_t* w_rt;  // 3x3 stride-1 only: "row-tap" weights [3*Cout][Kp_rt], row (s, o), col (r, c), or nullptr
  int Kp_rt;
  const float* bias;     // fp32 [Cout]
  const uint16_t* res;   // bf16 shortcut source, or nullptr
  const float* res32;    // fp32 shortcut source (fp32 residual stream), preferred when set
  uint16_t* y;           // bf16 [n][Ho][Wo][Cout]  (tensor-core operand copy)
  float* y32;            // fp32 [n][Ho][Wo][Cout]  (residual-stream copy) or nullptr
  const int* n_live;     // device live-row count (samples); nullptr -> n_static
  int n_static;
  int H, W, C, Ho, Wo, Cout, ksz, stride, pad;
  int K, Kp;
  int c_live = 0;       // input channels that can be nonzero (a prefix of C; 0 = all): the s4d stem's 48 of 64
  int relu;
  int res_mode;          // 0 none, 1 identity [n][Ho][Wo][Cout], 2 option A from [n][rH][rW][rC]
  int rH, rW, rC, r_pad_lo;
  int res_nhwc = 0;      // option-A bf16 shortcut tensor is NHWC (else channel-planar)
  int nhwc = 0;          // 1: bf16 output y and identity shortcut res are NHWC [n][H][W][C] (else channel-planar)
  int in_nhwc = 0;       // 1: bf16 input x is NHWC (the im2col GEMM); 0: channel-planar (planar kernels)
  // conv_gemm only: a second A operand concatenated along K (the fused projection shortcut of a
  // bottleneck block: D = conv1x1(x) + proj1x1/stride2(x2)); w is then [Cout][K + C2]
  const uint16_t* x2 = nullptr;   // bf16 NHWC [n][H2][W2][C2]
  int C2 = 0, H2 = 0, W2 = 0, stride2 = 1;
  // conv_gemm only, whole-sample tiles (128 % (Ho*Wo) == 0): sample i of the launch reads input
  // sample rows_in[i] (im2col path) and / or writes output (and identity-shortcut) sample
  // rows_out[i] -- the in-place form of a gate's then-branch; nullptr = dense order
  const int* rows_in = nullptr;
  const int* rows_out = nullptr;
  // conv_gemm only, zero-copy sub-network entry: the rows of the flat A operand
  // (a 1x1 / stride-1 conv) belong to input samples rows_gather[m / HW] -- loaded as boxes of
  // zero_copy_rows(HW, 64) rows at (pixel, sample) -- and the fused projection operand x2 to
  // samples x2_rows[m / HWo], loaded as im2col boxes of zero_copy_rows(HWo, 16) pixels; the
  // output stays dense
  const int* rows_gather = nullptr;
  const int* x2_rows = nullptr;
  // conv_gemm only (staged epilogue): fused GAP partials [M / gap_g][Cout] fp32 -- per group of
  // gap_g consecutive output rows (gap_g = the largest power of two <= 32 dividing Ho*Wo, so a
  // group never straddles samples and always covers the same pixels of its sample), the column
  // sums of y in ascending row order; see launch_gap_reduce
  float* gap_part = nullptr;
  int gap_g = 32;
  // dense rows only (Ho = Wo = 1): write y as a split pair [hi | lo] per row (row stride 2*Cout,
  // hi = bf16(v), lo = bf16(v - hi)) -- the operand format of the BF16X3 parity mode
  int split = 0;
  // dense rows only: fp32 output y32 with row stride y32_ld (0 = Cout) and only its first y32_n
  // columns stored (0 = all; a multiple of 4) -- the wide heads' padded-N GEMM writes the K
  // logits straight into the [rows][K] logit buffer
  int y32_ld = 0, y32_n = 0;
  // conv_gemm only: the "pair" residual stream -- y32 / res32 point to bf16 LO planes and the
  // stream value is bf16(hi) + bf16(lo) with hi = the bf16 operand copy (y / res) and
  // lo = bf16_rn(v - hi): 4 bytes per element instead of fp32 + bf16 copy (6), |rel err| < 2^-16
  int y32_pair = 0;
  // gemm_tma only: fused LM-head argmax.  Instead of storing y, each
  // epilogue thread scans its row's BN columns of the tile in ascending order (after bias, plus
  // the loop guard's EOS bias g_beta * (g_t + 1 - g_len[g_src[g_slot[m] * g_S]]) on column g_eos)
  // and writes the tile's (max, lowest index of the max) to am_val / am_idx [rows][Cout / BN]
  float* am_val = nullptr;
  int* am_idx = nullptr;
  const int32_t* g_slot = nullptr;
  const int32_t* g_src = nullptr;
  const float* g_len = nullptr;
  float g_beta = 0.f;
  int g_t = 0, g_S = 0, g_eos = -1;
  // gemm_tma only: residual + LayerNorm fused into the epilogue (the decoder's post-LN sub-layer
  // ends).  v = acc + bias + res32 (res_mode 1) is normalised over its whole row:
  // the N tiles of one M tile (BN = 64, same round of the persistent loop) publish per-row partial sums to
  // ln_part [rows][2][Cout / 64] and meet on ln_cnt[m_tile] (zero on entry, zero on exit) --
  // mean first, then the centred sum of squares, biased variance, eps; y32 <- LN(v) fp32 and
  // y <- bf16(LN(v)).  y32 may alias res32 (every element is read before it is written, by
  // the same thread)
  const float* ln_gamma = nullptr;
  const float* ln_beta = nullptr;
  float* ln_part = nullptr;
  int* ln_cnt = nullptr;
  float ln_eps = 0.f;
  // set by launch_gemm_tma: the N tiles of an M tile form one thread-block cluster and swap the
  // row partials through DSMEM (st.async into every peer's SMEM + an mbarrier) instead of L2
  int ln_cluster = 0;
  long long* ts = nullptr;   // development: conv_gemm phase timestamps (DYCL_TS_CONV)
  int dbg = 0;           // bit5 (32): row-tap mode opt-in; experiments only (results invalid): bit0 skip
                         // epilogue math/stores, bit1 skip MMAs, bit2 skip A loads, bit3 no residual prefetch.
                         // conv_gemm: 128 no staged epilogue, 256 no resident weights, 512 no tiled-shift
                         // A boxes (nor row-tap), 4194304 no row-tap; timing only: 1024 skip A loads,
                         // 2048 skip MMAs, 4096 skip the epilogue
};
// Programmatic dependent launch (PDL) for the launches the calling host thread enqueues
// while a PdlScope is alive (the config-4 decode loop: ~70 dependent small kernels per step).
// A PDL launch may start while its predecessor kernel is still running; every kernel that
// can be launched this way executes griddepcontrol.wait (ptx::pdl_wait / s2s pdl_wait)
// before its first read of predecessor output and before any early return, so completion
// stays transitive along the stream.  Thread-local: graphs are driven from several threads.
bool& pdl_flag();
struct PdlScope {
  bool prev;
  explicit PdlScope(bool on) : prev(pdl_flag()) { pdl_flag() = on; }
  ~PdlScope() { pdl_flag() = prev; }
};
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) for `func` on the CURRENT device, once per
// (device, function, size): function attributes are per device context, so a process that
// drives graphs on several devices must set them on each (thread-safe; hostmod.cu).
// One kernel of each translation unit's module (lazy-loading anchors, see preload_kernels).
const void* tu_anchor_conv_tc();
const void* tu_anchor_conv_tma();
const void* tu_anchor_conv_gemm();
const void* tu_anchor_conv_halo();
const void* tu_anchor_gemm_tma();
const void* tu_anchor_block_fused();
const void* tu_anchor_hostmod();
const void* tu_anchor_s2s_kernels();
const void* tu_anchor_cap();
const void* tu_anchor_drb();
// Load every kernel of libdycl now (CUDA lazy loading otherwise loads a kernel at its first
// launch, and loading can wait for the whole context to go idle: with device-initiated
// rebalancing between ranks of ONE process, a rank's spinning exchange kernel would then wait
// for a peer whose host thread is blocked loading its next kernel). Once per device.
cudaError_t preload_kernels();
cudaError_t ensure_smem(const void* func, size_t bytes);
template <typename... KArgs>
inline cudaError_t ensure_smem(void (*kernel)(KArgs...), size_t bytes) {
  return ensure_smem(reinterpret_cast<const void*>(kernel), bytes);
}
// Kernel launch honouring pdl_flag() (cudaLaunchKernelEx + programmatic stream serialization).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_flag() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Launch on `stream`; grid is sized for max_rows samples (persistent CTAs loop
// over the tiles the live count needs).  Returns cudaSuccess or the launch error.
cudaError_t launch_conv_tc(const ConvArgs& a, int max_rows, int num_sms, cudaStream_t stream);
// Row-tap weight layout for 3x3 / stride 1 / pad 1 convs: from the standard packed
// weights wp [cout][kp] (k = (r*3 + s)*cp + c) build [3*cout][kp_rt] with row s*cout + o,
// column r*cp + c (kp_rt = roundup(3*cp, 64)); the W taps then share one MMA (N = 3*cout).
inline void pack_rowtap(const uint16_t* wp, int cout, int kp, int cp, uint16_t* out, int kp_rt) {
  for (int s = 0; s < 3; ++s)
    for (int o = 0; o < cout; ++o) {
      uint16_t* row = out + ((size_t)s * cout + o) * kp_rt;
      for (int j = 0; j < kp_rt; ++j) row[j] = 0;
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < cp; ++c) row[r * cp + c] = wp[(size_t)o * kp + (size_t)(r * 3 + s) * cp + c];
    }
}
// TMA-fed variant (conv_tma.cu) for layers whose output tiles are rectangular
// boxes; *handled = false (and nothing launched) when the shape does not qualify.
cudaError_t launch_conv_tma(const ConvArgs& a, int max_rows, int num_sms, cudaStream_t stream, bool* handled);
// Dense-layer GEMM on tcgen05 with TMA SWIZZLE_128B tiles (gemm_tma.cu): [rows][K] x [N][K].
// 3x3 / 4x4 stride-1 NHWC conv, 64 -> 64 / 128 / 256 or 16 -> 64 channels, whole output rows per
// 128-row tile, bf16 output only: TMA halo tile + shifted UMMA descriptors (conv_halo.cu)
bool conv_halo_eligible(const ConvArgs& a);
cudaError_t launch_conv_halo(const ConvArgs& a, int max_rows, int num_sms, cudaStream_t stream);
bool gemm_tma_eligible(const ConvArgs& a);
cudaError_t launch_gemm_tma(const ConvArgs& a, int max_rows, int num_sms, cudaStream_t stream);
// N tile width launch_gemm_tma picks for these arguments (64, 128 or 256).
int gemm_tma_bn(const ConvArgs& a, int max_rows, int num_sms);
// The fused residual + LayerNorm epilogue (ConvArgs.ln_*) applies: BN = 64, d / 64 <= 16 N tiles.
bool gemm_tma_ln_ok(const ConvArgs& a, int max_rows, int num_sms);

// NHWC implicit-GEMM conv with TMA im2col operand loads (conv_gemm.cu): C % 64 == 0, Cout % 64 == 0.
bool conv_gemm_eligible(const ConvArgs& a);
// Zero-copy entry box height for samples of `hw` rows: the largest power of two <= cap that
// divides hw (a box then never straddles two samples); usable when >= ZC_MIN_ROWS (56x56: 64,
// 28x28: 16, 14x14: 4; 7x7: 1, not usable).
constexpr int ZC_MIN_ROWS = 4;
inline int zero_copy_rows(int hw, int cap) {
  const int g = hw & -hw;
  return g < cap ? g : cap;
}
cudaError_t launch_conv_gemm(const ConvArgs& a, int max_rows, int num_sms, cudaStream_t stream);
// Dispatch: path 0 = auto (TMA when possible), 1 = cp.async kernel, 2 = TMA only.
cudaError_t launch_conv(const ConvArgs& a, int max_rows, int num_sms, cudaStream_t stream, int path = 0);

// a0: fp32 [n][HW][C] -> bf16 [n][HW][Cp]  (Cp = roundup(C, 8), zero pad)
cudaError_t launch_cast_pad(const float* in, uint16_t* out, int64_t n, int hw, int c, int cp,
                            cudaStream_t s);

// pooled[n][c] = (sum over the HW / G row groups k = 0.. of sample n of gap_part[n*HW/G + k][c],
// in ascending k) / HW -- a fixed order, independent of the sample's batch position.
cudaError_t launch_gap_reduce(const float* gap_part, int G, float* pooled, const int* n_live, int max_rows, int HW, int C,
                              cudaStream_t s);

// a0 for a space-to-depth stem: fp32 NHWC [n][H][W][c] -> bf16 [n][H/4][W/4][64], channel
// (pr*4 + ps)*c + ci = input pixel (4P+pr, 4Q+ps) channel ci; channels >= 16c zero (c <= 4).
cudaError_t launch_cast_s4d(const float* in, uint16_t* out, int64_t n, int H, int W, int c, cudaStream_t s);
// a0 for the 2x2 space-to-depth stem: fp32 [n][H][W][c] (c <= 4) -> bf16 [n][H/2][W/2][16],
// channel (dy*2+dx)*c + ci, zero-padded to 16
cudaError_t launch_cast_s2d2(const float* in, uint16_t* out, int64_t n, int H, int W, int c, cudaStream_t s);

// Run-start init: counts[0] = n ; orig[i] = i ; path[i] = 0.
cudaError_t launch_init(int* counts, int n, int* orig, int32_t* path, float* margin, int nmax, cudaStream_t s);
// a9 survivor rebalancing (hostmod.cu): pack the metadata of rows leaving the rank, unpack the
// rows that arrived, scatter returned results home by id, set a device count
cudaError_t launch_rb_pack(const int* orig, int first, int n, const int32_t* res_path, const float* res_margin,
                           const long long* ext_gid, long long gid_base, int batch, int* sent_orig, int32_t* meta,
                           cudaStream_t s);
cudaError_t launch_rb_unpack(int* orig, int first, int n, int ext0, int batch, const int32_t* meta,
                             int32_t* res_path, float* res_margin, long long* ext_gid, cudaStream_t s);
cudaError_t launch_rb_return(const int* sent_orig, int n, int K, const float* ret_logits, const int32_t* ret_path,
                             const float* ret_margin, float* res_logits, int32_t* res_path, float* res_margin,
                             cudaStream_t s);
cudaError_t launch_set_int(int* p, int v, cudaStream_t s);

// GAP + FC head + predicate, one CTA per live sample.
//   kind 0 = exit (flag = max softmax >= thr), 1 = gate (flag = sigmoid(z0) > thr), 2 = final (flag = 1)
struct HeadArgs {
  const uint16_t* h;     // bf16 [n][HW][C]   (used when h32 == nullptr)
  const float* h32;      // fp32 [n][HW][C]   residual stream
  const uint16_t* w;     // bf16 [K][C]
  const float* b;        // fp32 [K]
  float* z;              // fp32 [n][K] logits scratch
  uint8_t* flag;         // [n]
  float* pred;           // [n] predicate value (conf or p) for diagnostics, may be null
  const int* n_live;
  int HW, C, K, kind;
  float thr;
  int nhwc = 0;          // bf16 h is NHWC [n][HW][C] (else channel-planar)
  // wide heads (K >= 128): FC batched over FC_ROWS samples per CTA from the transposed weights
  const uint16_t* wt = nullptr;   // bf16 [C][K] (nullptr: per-sample FC inside the GAP kernel)
  const float* pooled = nullptr;  // fp32 [rows][C] pooled features already computed (fused GAP): skip the GAP
  float* pooled_out = nullptr;    // fp32 [rows][C]: keep the GAP this kernel computes (later in-place gates reuse it)
  float* gpool = nullptr;         // fp32 [rows][C] pooled-feature scratch for the batched FC
  int h32_pair = 0;               // h32 is the pair stream's bf16 lo plane (value = h + lo), NHWC
  // wide heads on the tensor cores (a2): the fp32 pooled features are split into a bf16 pair
  // [hi | lo] per row (a2, [rows][2C]) and multiplied with w2 = [W | W] ([kpad][2C], rows >= K
  // zero) by the tcgen05 GEMM -- the split-bf16 product, fp32-accurate (|rel err| ~ 2^-16)
  // because the weights are exact bf16 -- writing the K logits to z; b2 = bias padded to kpad
  const uint16_t* w2 = nullptr;
  const float* b2 = nullptr;
  uint16_t* a2 = nullptr;
  int kpad = 0, num_sms = 148;
};
cudaError_t launch_head(const HeadArgs& a, int max_rows, cudaStream_t s);

// Recurrent gate (SkipNet RNN gate): per live row r, u = u[r][0..n_in) (the proj head's fp32
// output), state = state[orig[r]] (h [H] then c [H], fp32); LSTM cell step (torch gate order
// i, f, g, o; w = w_ih [4H][n_in] | w_hh [4H][H] | b_ih [4H] | b_hh [4H]); the new state is
// written back; z = w_out . h + b_out, p = sigmoid(z), flag = p > thr, pred = p.  Warp per row.
struct RnnGateArgs {
  const float* u;
  int u_stride;
  const int* orig;
  float* state;
  const float* w;
  const float* w_out;
  float b_out;
  int n_in, hidden;
  float thr;
  uint8_t* flag;
  float* pred;
  const int* n_live;
};
cudaError_t launch_rnn_gate(const RnnGateArgs& a, int max_rows, int num_sms, cudaStream_t s);

// Stable partition of the live rows by flag (single CTA, deterministic):
//   rows with flag==1 -> list1 (in order), count -> counts_out[0]
//   rows with flag==0 -> list0 (in order), count -> counts_out[1]
//   orig_next = [orig[list0...]]  (mode 0: survivors continue; exit)
//             = [orig[list1...], orig[list0...]]  (mode 1: gate; then-rows first)
//   mode 1 also ORs path_bit into path[orig[i]] for flag==1 rows.
//   margin (optional): margin[orig[i]] = min(margin[orig[i]], |pred[i] - thr|), the per-sample
//   distance of its predicates from their thresholds along its path (band reporting, R12).
cudaError_t launch_compact(const uint8_t* flag, const int* n_live, const int* orig,
                           int* list1, int* list0, int* counts_out, int* orig_next,
                           int mode, int32_t* path, int32_t path_bit, const float* pred, float thr, float* margin,
                           cudaStream_t s);

// out_logits[orig[list[j]]] = z[list[j]], out_path[orig[list[j]]] = path_val (if path_val >= 0)
// for j < *count.
cudaError_t launch_scatter(const float* z, int K, const int* list, const int* count, const int* orig,
                           float* out_logits, int32_t* out_path, int32_t path_val, int max_rows,
                           cudaStream_t s);

// dst row (dst_off + j) = transform(src row list[j]) for j < *count.
//   mode 0: identity copy of row_bytes (multiple of 16)
//   mode 1: option A: src [H][W][C] -> dst [H/2][W/2][2C] subsample + zero pad (C/2 each side)
// dst_off_count: if non-null, rows are written from offset *dst_off_count.
struct GatherArgs {
  const void* src;
  void* dst;
  int elem_bytes;          // 2 (bf16) or 4 (fp32)
  const int* list;
  const int* count;
  const int* dst_off_count;
  int64_t row_elems_src;   // elements per src row
  int64_t row_elems_dst;
  int mode, H, W, C;
  int dst_nhwc = 0;        // mode 1, bf16: destination NHWC (else channel-planar)
};
cudaError_t launch_gather(const GatherArgs& a, int max_rows, int num_sms, cudaStream_t s);

// Max pooling (k x k, stride, pad) of a tensor pair: input fp32 NHWC (x32) if given,
// else bf16 channel-planar (x); output bf16 channel-planar (y) and fp32 NHWC (y32, optional).
struct PoolArgs {
  const uint16_t* x;
  const float* x32;
  uint16_t* y;
  float* y32;
  const int* n_live;
  int H, W, C, Ho, Wo, k, stride, pad;
  int nhwc = 0;          // bf16 x / y are NHWC (else channel-planar)
  int s2d = 0;           // 3x3/2/1 pool over a 2x2-phase input [n][Ho][Wo][4C] (channel (b*2+b')*C + c
                         // = pixel (2ho+b, 2wo+b')); output NHWC [n][Ho][Wo][C]
};
cudaError_t launch_maxpool(const PoolArgs& a, int max_rows, int num_sms, cudaStream_t s);

// Fused residual basic blocks (block_fused.cu): nblk consecutive blocks y = relu(conv2(relu(conv1(x)))
// + x), 3x3 / stride 1, whole sample per CTA iteration kept in SMEM across the blocks, fp32 stream
// in/out (+ optional bf16 channel-planar copy of the last block's output).
constexpr int MAX_FUSED_BLOCKS = 8;
struct BlockArgs {
  const float* x32;        // fp32 NHWC [n][H][W][C] (the first block's input, also its shortcut)
  const int32_t* list;     // optional row index list (input row = list[i]), nullptr = identity
  int list_out = 0;        // 1: output row = list[i] too (in place over x when y32 == x32)
  float* pooled = nullptr; // fp32 [rows][C]: per-sample channel means of the last block's y (fused GAP), or nullptr
  float* y32;              // fp32 NHWC [n][H][W][C]
  uint16_t* yb;            // bf16 channel-planar copy or nullptr
  int nblk;                // blocks fused in this launch (1..MAX_FUSED_BLOCKS)
  const uint16_t* w1_rt[MAX_FUSED_BLOCKS];   // row-tap weights [3C][Kp_rt] (pack_rowtap) per block
  const uint16_t* w2_rt[MAX_FUSED_BLOCKS];
  const float* b1[MAX_FUSED_BLOCKS];
  const float* b2[MAX_FUSED_BLOCKS];
  const int* n_live;
  int n_static, C, H, W;
  long long* ts;           // debug only: per-phase clock64 stamps of CTA 0 (nullptr = off)
};
bool block_fused_eligible(int C, int H, int W);
cudaError_t launch_block_fused(const BlockArgs& a, int max_rows, int num_sms, cudaStream_t stream);

}  // namespace dycl
