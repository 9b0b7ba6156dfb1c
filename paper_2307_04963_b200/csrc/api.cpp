// libdycl runtime: C ABI (include/dycl.h), restricted-HCFG registry, Alg.-2-style
// shape propagation and buffer planning, and the device-side plan executor.
//
// PAPER.md mapping:
//   sub-network   = HCFG tensor node, conditional-free (Sec. 5.3)
//   exit / gate   = HCFG logic node evaluated on an intermediate tensor (L265)
//   finalize      = Alg. 2 (L658-716): walk the chain from N0 carrying the shape;
//                   a logic node's output shape is its predecessor's; each tensor
//                   node is "compiled" (planned) for the predecessor's output shape
//   run           = the host API P_Host(x) (Sec. 5.6) -- but enqueued as
//                   device work only: predicates, compaction and scatter are
//                   kernels, the live counts stay in HBM (Challenge 2, L499-501).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/dycl.h"
#include "comm.h"
#include "drb.h"
#include "kernels.h"

namespace {

struct Shape {
  int H = 0, W = 0, C = 0;   // C = logical channels
  int Cp() const { return (C + 7) / 8 * 8; }
  bool operator==(const Shape& o) const { return H == o.H && W == o.W && C == o.C; }
  long long row_elems() const { return (long long)H * W * Cp(); }
};

enum LayerKind { L_CONV, L_DENSE, L_GAP, L_BLOCK, L_MAXPOOL, L_PROJ };

struct Layer {
  LayerKind kind;
  int cout = 0, k = 1, stride = 1, pad = 0, relu = 0, residual = 0, out_fp32 = 0;
  std::vector<uint16_t> w;
  std::vector<float> b;
  // planned at finalize
  Shape in, out;
  int K = 0, Kp = 0, res_mode = 0;
  Shape res_shape;
  uint16_t* d_w = nullptr;
  uint16_t* d_wrt = nullptr;    // row-tap layout (3x3 / stride 1 / pad 1 convs)
  int Kp_rt = 0;
  float* d_b = nullptr;
  // space-to-depth stem (NHWC graphs): a 7x7 / stride-2 conv on <= 4 channels runs as a 3x3 /
  // stride-1 conv over 4x4 pixel blocks (64 channels) producing the 2x2 output phases as
  // 4*cout channels; d_w / d_b then hold that packed form ([4*cout][9*64], [4*cout])
  int s4d = 0;
  int pool_s2d = 0;           // maxpool reading that phase layout (3x3 / stride 2 / pad 1)
  // 2x2 space-to-depth stem (opt-in, measured slower than s4d): the 7x7 / stride-2 conv on <= 4 channels as a 4x4 /
  // stride-1 conv over 2x2 pixel blocks (16 channels) with padding 2 before / 1 after, on the
  // halo-tile kernel (conv_halo.cu); d_w holds [cout][16 taps x 16] ; output plain NHWC
  int s2d2 = 0;
  uint16_t* d_wt = nullptr;   // wide fp32 heads (K >= 128): weights transposed [C][K] for the batched FC
  uint16_t* d_w2 = nullptr;   // wide fp32 heads on the tensor cores: [W | W] [kpad][2C] (split-bf16 GEMM)
  float* d_b2 = nullptr;      // bias padded to kpad
  int kpad = 0;
  // NHWC bottleneck: this 1x1 conv and the projection shortcut before it run as ONE GEMM over
  // K-concatenated operands [t | x] with weights [W | W_proj] and bias b + b_proj
  int fuse_proj = 0;
  uint16_t* d_wcat = nullptr;
  float* d_bcat = nullptr;
};

struct Subnet {
  std::vector<Layer> layers;
  bool ended = false;
  bool is_head = false;       // [GAP] + dense(out_fp32)
  Shape in, out;
  int head_K = 0;
  bool needs_in32 = true;     // reads its input's fp32 residual-stream copy (set at finalize)
};

enum NodeKind { N_SEQ, N_EXIT, N_GATE, N_FINAL };
struct Node {
  NodeKind kind;
  int sn = -1, then_sn = -1;
  float thr = 0.f;
  int ordinal = 0;            // exit index / gate index
  int skip_mode = 0;          // gate: 0 identity, 1 option A
  Shape in, out;
  // recurrent gate (dycl_gate_rnn): the proj subnet yields the cell input u; the graph's LSTM cell
  // steps on it; z = w_out . h + b_out
  int rnn = 0;
  std::vector<float> w_out;
  float b_out = 0.f;
  float* d_w_out = nullptr;
};

struct Launch {               // profiling record
  int kind;
  cudaEvent_t e0, e1;
  const int* count_dev;       // live-count slot the launch processed
  double bytes_per_row, flops_per_row, bytes_fixed;
};

}  // namespace

struct dycl_graph_s {
  int device = 0;
  Shape input;
  std::vector<Subnet> subnets;
  std::vector<Node> nodes;
  bool finalized = false;
  int64_t max_batch = 0;
  int num_sms = 148;
  int K = 0;
  int n_exits = 0, n_gates = 0;
  std::string err;
  // the recurrent gates' shared LSTM cell (dycl_rnn_cell) and its per-sample state [max_batch][2H]
  int rnn_in = 0, rnn_hidden = 0;
  std::vector<float> rnn_w;            // w_ih [4H][n_in] | w_hh [4H][H] | b_ih [4H] | b_hh [4H]
  float* d_rnn_w = nullptr;
  float* d_rnn_state = nullptr;
  // device workspace
  static constexpr int NBUF = 6;
  static constexpr int NBUF32 = 4;
  uint16_t* buf[NBUF] = {};
  float* buf32[NBUF32] = {};
  int precision = DYCL_PREC_FP32_STREAM;
  int conv_path = 0;                 // 0 auto; DYCL_CONV_PATH=1 forces the cp.async kernel
  int conv_dbg = 0;                  // DYCL_CONV_DBG: timing experiments only (results invalid)
  int halo_kskip = 1;                // DYCL_HALO_KSKIP=0: the s4d stem multiplies its zero channels too
  int no_fuse = 0;                   // DYCL_NO_FUSE=1: run basic blocks as two conv launches
  int head_cuda_core = 0;            // DYCL_HEAD_CUDA_CORE=1: wide-head FC on CUDA cores (k_head_fc), not tcgen05
  // pair residual stream (set at finalize; DYCL_NO_PAIR=1 disables): in NHWC graphs without gates,
  // fused blocks or dense trunk layers the fp32 stream copy is replaced by a bf16 "lo" plane
  // (value = bf16 operand copy + lo; ConvArgs::y32_pair): 4 instead of 6 bytes per element
  bool stream_pair = false;
  int max_fuse = dycl::MAX_FUSED_BLOCKS;   // DYCL_MAX_FUSE: basic blocks per fused launch (1..8)
  int no_inplace = 0;                // DYCL_NO_INPLACE=1: gates gather / merge instead of running in place
  int no_zero_copy = 0;              // DYCL_NO_ZERO_COPY=1: exits gather survivors even before a fused block
  int zc_proj_min = 8;               // smallest projection box (pixels) of a zero-copy GEMM entry (DYCL_ZC_PROJ_MIN)
  // CUDA graph of a whole run, captured on first use per (io pointers, batch) and replayed;
  // every kernel sizes itself from device counts, so the captured launch sequence is valid for
  // any data (DYCL_GRAPH=0 disables; profiling runs are issued launch by launch)
  bool use_graph = true;
  cudaStream_t cap_stream = nullptr;
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    const void* key[4] = {};
    int64_t batch = -1;
    long long goff = -1;             // device-rebalanced runs: the global offset baked into the graph
    int launches = 0;
    uint64_t used = 0;
  };
  static constexpr int NGRAPH = 4;   // dycl_run_host alternates staging slots and a tail chunk
  GraphEntry graphs[NGRAPH];
  uint64_t graph_clock = 0;
  // dycl_run_host pipeline: H2D of sub-chunk k+1 and D2H of k-1 overlap the run of k
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  cudaEvent_t ev_h2d[2] = {}, ev_run[2] = {}, ev_d2h[2] = {};
  int nhwc = 0;                      // bf16 activations NHWC (decided at finalize; DYCL_NHWC=0 disables)
  int stem_s4d = 0;                  // input cast to 4x4 space-to-depth for the stem (DYCL_STEM_S4D=0 disables)
  int stem_s2d2 = 0;                 // input cast to 2x2 space-to-depth, 16 channels (opt-in DYCL_STEM_S2D2=1)
  long long* dbg_ts = nullptr;       // DYCL_TS=1: fused-block phase timestamps (development)
  int dbg_ts_conv = 0;               // DYCL_TS_CONV=k: record conv_gemm phases of the k-th conv launch
  int dbg_ts_pick = 0;               // DYCL_TS=k > 1: record the k-th fused launch of a run (else the last)
  long long max_row_elems = 0;
  int* d_counts = nullptr;
  int n_slots = 0;
  int* d_orig[2] = {};
  int* d_list1 = nullptr;
  int* d_list0 = nullptr;
  uint8_t* d_flag = nullptr;
  float* d_pred = nullptr;
  float* d_z = nullptr;
  float* d_gpool = nullptr;         // pooled features of wide heads [max_batch][max head C]
  uint16_t* d_a2 = nullptr;         // their split bf16 pairs [max_batch][2 * max head C] (tensor-core heads)
  float* d_gap_part = nullptr;      // conv_gemm fused-GAP partials [rows / G][C] fp32 (sub-network outputs read by a head)
  float* d_gap_pooled = nullptr;    // their reduction [max_batch][C]
  float* d_pool32[NBUF32] = {};     // fused-GAP features per fp32 stream buffer [max_batch][<= 32] (fused blocks)
  float* d_in_stage = nullptr;      // dycl_run_host staging (stage_rows rows)
  int64_t stage_rows = 0;
  float* d_logit_stage = nullptr;
  int32_t* d_path_stage = nullptr;
  float* d_margin_stage = nullptr;
  int launches_per_run = 0;
  // profiling
  bool profiling = false;
  std::vector<Launch> prof;
  size_t prof_used = 0;
  cudaStream_t prof_stream = nullptr;
  // multi-GPU survivor rebalancing (dycl_set_comm / dycl_set_comm_local)
  dycl::Transport* tr = nullptr;
  int rb_policy = 0;                 // bit k: rebalance after exit k (-1: every exit)
  // result space of a rebalancing run: rows [0, batch) are the rank's own samples, rows
  // [batch, batch + ext) the samples other ranks handed over (returned to them at the end)
  float* d_res_logits = nullptr;
  int32_t* d_res_path = nullptr;
  float* d_res_margin = nullptr;
  long long* d_ext_gid = nullptr;
  int* d_sent_orig = nullptr;        // result-space ids of the rows sent away, per level
  int32_t* d_meta = nullptr;         // [rows][4] path, margin bits, global id lo / hi (send | recv)
  float* d_ret_logits = nullptr;     // returned results of rows sent away
  int32_t* d_ret_path = nullptr;
  float* d_ret_margin = nullptr;
  int64_t rb_rows = 0;               // capacity of the result space / sent tables (rows)
  long long rb_sent = 0, rb_recv = 0;   // rows moved by the last run (dycl_rebalance_stats)
  // device-initiated rebalancing (dycl_set_rebalance_mode DEVICE; drb.cu)
  bool rb_device = false;
  void* drb_win = nullptr;           // this rank's window (transport-owned)
  void** drb_peers = nullptr;        // device [world] window bases
  size_t drb_bytes = 0, drb_rows_off = 0, drb_ret_off = 0;
  dycl::DrbPlan* d_drb_plan = nullptr;
  unsigned* d_drb_epoch = nullptr;
  int* d_drb_err = nullptr;
  int* d_drb_ticket = nullptr;
  int drb_levels_last = 0;           // levels the last run rebalanced (stats)
};

static thread_local std::string g_create_err;

namespace {

dycl_status fail(dycl_graph g, dycl_status s, const std::string& msg) {
  if (g) g->err = msg; else g_create_err = msg;
  return s;
}
dycl_status cuda_fail(dycl_graph g, cudaError_t e, const char* where) {
  return fail(g, DYCL_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define CK(call)                                            \
  do {                                                      \
    cudaError_t e_ = (call);                                \
    if (e_ != cudaSuccess) return cuda_fail(g, e_, #call);  \
  } while (0)

dycl_status check_sn(dycl_graph g, dycl_node sn) {
  if (!g) return DYCL_E_INVALID_ARG;
  if (g->finalized) return fail(g, DYCL_E_STATE, "graph already finalized");
  if (sn < 0 || sn >= (int)g->subnets.size()) return fail(g, DYCL_E_INVALID_ARG, "bad subnet id");
  if (g->subnets[sn].ended) return fail(g, DYCL_E_STATE, "subnet already ended");
  return DYCL_OK;
}

template <typename T>
dycl_status dmalloc(dycl_graph g, T** p, size_t bytes) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), bytes);
  if (e != cudaSuccess) return fail(g, DYCL_E_OOM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  return DYCL_OK;
}

// Fused-GAP row group: the largest power of two <= 32 dividing the per-sample pixel count
// (a group then never straddles samples; see ConvArgs::gap_g).
int gap_group(int hw) {
  int G = 32;
  while (G > 1 && hw % G) G >>= 1;
  return G;
}

// Shape propagation through one subnet (Alg. 2 line: "compile N with the shape of
// its predecessor").  Fills each layer's in/out and packed-weight geometry.
dycl_status plan_subnet(dycl_graph g, Subnet& s, const Shape& in, int sn_id) {
  Shape cur = in;
  Shape block_src;
  bool have_block = false;
  s.in = in;
  for (size_t li = 0; li < s.layers.size(); ++li) {
    Layer& L = s.layers[li];
    L.in = cur;
    char where[96];
    snprintf(where, sizeof where, "subnet %d layer %zu: ", sn_id, li);
    switch (L.kind) {
      case L_BLOCK:
        block_src = cur;
        have_block = true;
        L.out = cur;
        break;
      case L_GAP:
        L.out = Shape{1, 1, cur.C};
        cur = L.out;
        break;
      case L_MAXPOOL: {
        const int Ho = (cur.H + 2 * L.pad - L.k) / L.stride + 1;
        const int Wo = (cur.W + 2 * L.pad - L.k) / L.stride + 1;
        if (Ho <= 0 || Wo <= 0 || cur.C % 8) return fail(g, DYCL_E_SHAPE_MISMATCH, std::string(where) + "maxpool shape");
        L.out = Shape{Ho, Wo, cur.C};
        cur = L.out;
        break;
      }
      case L_PROJ: {
        if (!have_block) return fail(g, DYCL_E_SHAPE_MISMATCH, std::string(where) + "projection without block_begin");
        L.in = block_src;
        if ((int)L.w.size() != L.cout * block_src.C)
          return fail(g, DYCL_E_SHAPE_MISMATCH, std::string(where) + "projection c_in disagrees with the saved tensor");
        L.out = Shape{(block_src.H - 1) / L.stride + 1, (block_src.W - 1) / L.stride + 1, L.cout};
        L.K = block_src.Cp();
        L.Kp = (L.K + 63) / 64 * 64;
        block_src = L.out;            // the projection is now the shortcut
        break;
      }
      case L_CONV: {
        if ((int)L.w.size() != L.cout * L.k * L.k * cur.C)
          return fail(g, DYCL_E_SHAPE_MISMATCH, std::string(where) + "conv weight size != c_out*k*k*c_in");
        const int Ho = (cur.H + 2 * L.pad - L.k) / L.stride + 1;
        const int Wo = (cur.W + 2 * L.pad - L.k) / L.stride + 1;
        if (Ho <= 0 || Wo <= 0) return fail(g, DYCL_E_SHAPE_MISMATCH, std::string(where) + "empty output");
        L.out = Shape{Ho, Wo, L.cout};
        L.K = L.k * L.k * cur.Cp();
        L.Kp = (L.K + 63) / 64 * 64;
        L.res_mode = 0;
        if (L.residual) {
          if (!have_block) return fail(g, DYCL_E_SHAPE_MISMATCH, std::string(where) + "residual without block_begin");
          L.res_shape = block_src;
          if (block_src == L.out) L.res_mode = 1;
          else if (block_src.H == 2 * Ho && block_src.W == 2 * Wo && 2 * block_src.C == L.cout &&
                   block_src.C % 16 == 0)
            L.res_mode = 2;
          else return fail(g, DYCL_E_SHAPE_MISMATCH, std::string(where) + "shortcut shape neither identity nor option A");
        }
        cur = L.out;
        break;
      }
      case L_DENSE: {
        if (cur.H != 1 || cur.W != 1)
          return fail(g, DYCL_E_SHAPE_MISMATCH, std::string(where) + "dense needs a [1][1][C] input (add gap)");
        if ((int)L.w.size() != L.cout * cur.C)
          return fail(g, DYCL_E_SHAPE_MISMATCH, std::string(where) + "dense weight size != n_out*n_in");
        L.out = Shape{1, 1, L.cout};
        if (L.out_fp32) {
          if (li + 1 != s.layers.size())
            return fail(g, DYCL_E_SHAPE_MISMATCH, std::string(where) + "fp32 head must be the last layer");
        } else {
          L.K = cur.Cp();
          L.Kp = (L.K + 63) / 64 * 64;
        }
        cur = L.out;
        break;
      }
    }
  }
  s.out = cur;
  // head pattern: [gap] dense(out_fp32)
  s.is_head = false;
  const size_t n = s.layers.size();
  if (n >= 1 && s.layers[n - 1].kind == L_DENSE && s.layers[n - 1].out_fp32) {
    if (n == 1 || (n == 2 && s.layers[0].kind == L_GAP)) {
      s.is_head = true;
      s.head_K = s.layers[n - 1].cout;
    } else {
      return fail(g, DYCL_E_UNSUPPORTED, "fp32 heads must be [gap] + dense(out_fp32)");
    }
  }
  return DYCL_OK;
}

dycl_status upload_subnet(dycl_graph g, Subnet& s) {
  for (size_t li = 0; li < s.layers.size(); ++li) {
    Layer& L = s.layers[li];
    if (g->nhwc && L.kind == L_CONV && li > 0 && s.layers[li - 1].kind == L_PROJ && L.k == 1 && L.stride == 1 &&
        L.res_mode == 1 && L.in.C % 64 == 0 && s.layers[li - 1].in.C % 64 == 0 && !getenv("DYCL_NO_FUSE_PROJ")) {
      const Layer& Pj = s.layers[li - 1];
      const int K1 = L.in.C, K2 = Pj.in.C, co = L.cout;
      std::vector<uint16_t> wc((size_t)co * (K1 + K2));
      std::vector<float> bc(co);
      for (int o = 0; o < co; ++o) {
        for (int c = 0; c < K1; ++c) wc[(size_t)o * (K1 + K2) + c] = L.w[(size_t)o * K1 + c];
        for (int c = 0; c < K2; ++c) wc[(size_t)o * (K1 + K2) + K1 + c] = Pj.w[(size_t)o * K2 + c];
        bc[o] = L.b[o] + Pj.b[o];
      }
      dycl_status st = dmalloc(g, &L.d_wcat, wc.size() * 2);
      if (st) return st;
      CK(cudaMemcpy(L.d_wcat, wc.data(), wc.size() * 2, cudaMemcpyHostToDevice));
      if ((st = dmalloc(g, &L.d_bcat, bc.size() * 4))) return st;
      CK(cudaMemcpy(L.d_bcat, bc.data(), bc.size() * 4, cudaMemcpyHostToDevice));
      L.fuse_proj = 1;
    }
    if (L.kind == L_CONV && L.s2d2) {
      // W'[o][(R*4+S)*16 + (dy*2+dx)*Cin + c] = w[o][2R+dy-1][2S+dx-1][c] (zero outside the 7x7
      // window): output pixel y reads input rows 2y-3 .. 2y+3 = blocks y-2 .. y+1 (tap R = block - y + 2)
      const int Cin = L.in.C, co = L.cout, K2 = 16 * 16;
      std::vector<uint16_t> w2((size_t)co * K2, 0);
      for (int o = 0; o < co; ++o)
        for (int R = 0; R < 4; ++R)
          for (int S = 0; S < 4; ++S)
            for (int dy = 0; dy < 2; ++dy)
              for (int dx = 0; dx < 2; ++dx) {
                const int r = 2 * R + dy - 1, s2 = 2 * S + dx - 1;
                if (r < 0 || r >= L.k || s2 < 0 || s2 >= L.k) continue;
                for (int c = 0; c < Cin; ++c)
                  w2[(size_t)o * K2 + (R * 4 + S) * 16 + (dy * 2 + dx) * Cin + c] =
                      L.w[(((size_t)o * L.k + r) * L.k + s2) * Cin + c];
              }
      dycl_status st = dmalloc(g, &L.d_w, w2.size() * 2);
      if (st) return st;
      CK(cudaMemcpy(L.d_w, w2.data(), w2.size() * 2, cudaMemcpyHostToDevice));
      if ((st = dmalloc(g, &L.d_b, L.b.size() * 4))) return st;
      CK(cudaMemcpy(L.d_b, L.b.data(), L.b.size() * 4, cudaMemcpyHostToDevice));
      continue;
    }
    if (L.kind == L_CONV && L.s4d) {
      // W'[(b*2+b')*cout + o][(R*3+S)*64 + (pr*4+ps)*Cin + c] = w[o][r][s][c] with
      // r = 4(R-1) + pr - 2b + pad, s = 4(S-1) + ps - 2b' + pad (zero outside the 7x7 window):
      // output pixel (2P+b, 2Q+b') reads input rows 4(P+R-1)+pr of blocks P-1..P+1.
      const int Cin = L.in.C, co = L.cout, K4 = 9 * 64;
      std::vector<uint16_t> w4((size_t)4 * co * K4, 0);
      for (int b = 0; b < 2; ++b)
        for (int b2 = 0; b2 < 2; ++b2)
          for (int o = 0; o < co; ++o)
            for (int R = 0; R < 3; ++R)
              for (int S = 0; S < 3; ++S)
                for (int pr = 0; pr < 4; ++pr)
                  for (int ps = 0; ps < 4; ++ps) {
                    const int r = 4 * (R - 1) + pr - 2 * b + L.pad, s2 = 4 * (S - 1) + ps - 2 * b2 + L.pad;
                    if (r < 0 || r >= L.k || s2 < 0 || s2 >= L.k) continue;
                    for (int c = 0; c < Cin; ++c)
                      w4[(size_t)((b * 2 + b2) * co + o) * K4 + (R * 3 + S) * 64 + (pr * 4 + ps) * Cin + c] =
                          L.w[(((size_t)o * L.k + r) * L.k + s2) * Cin + c];
                  }
      dycl_status st = dmalloc(g, &L.d_w, w4.size() * 2);
      if (st) return st;
      CK(cudaMemcpy(L.d_w, w4.data(), w4.size() * 2, cudaMemcpyHostToDevice));
      std::vector<float> b4((size_t)4 * co);
      for (int q = 0; q < 4; ++q)
        for (int o = 0; o < co; ++o) b4[(size_t)q * co + o] = L.b[o];
      if ((st = dmalloc(g, &L.d_b, b4.size() * 4))) return st;
      CK(cudaMemcpy(L.d_b, b4.data(), b4.size() * 4, cudaMemcpyHostToDevice));
      continue;
    }
    if (L.kind == L_CONV || L.kind == L_PROJ || (L.kind == L_DENSE && !L.out_fp32)) {
      // repack to [Cout][k][k][Cp] padded along K to Kp (zeros)
      const int Cin = L.in.C, Cp = L.in.Cp();
      std::vector<uint16_t> wp((size_t)L.cout * L.Kp, 0);
      for (int o = 0; o < L.cout; ++o)
        for (int t = 0; t < L.k * L.k; ++t)
          for (int c = 0; c < Cin; ++c)
            wp[(size_t)o * L.Kp + (size_t)t * Cp + c] = L.w[((size_t)o * L.k * L.k + t) * Cin + c];
      dycl_status st = dmalloc(g, &L.d_w, wp.size() * 2);
      if (st) return st;
      CK(cudaMemcpy(L.d_w, wp.data(), wp.size() * 2, cudaMemcpyHostToDevice));
      if (L.kind == L_CONV && L.k == 3 && L.stride == 1 && L.pad == 1) {
        L.Kp_rt = (3 * Cp + 63) / 64 * 64;
        std::vector<uint16_t> wr((size_t)3 * L.cout * L.Kp_rt);
        dycl::pack_rowtap(wp.data(), L.cout, L.Kp, Cp, wr.data(), L.Kp_rt);
        if ((st = dmalloc(g, &L.d_wrt, wr.size() * 2))) return st;
        CK(cudaMemcpy(L.d_wrt, wr.data(), wr.size() * 2, cudaMemcpyHostToDevice));
      }
    } else if (L.kind == L_DENSE) {
      const int Cin = L.in.C, Cp = L.in.Cp();
      std::vector<uint16_t> wp((size_t)L.cout * Cp, 0);
      for (int o = 0; o < L.cout; ++o)
        for (int c = 0; c < Cin; ++c) wp[(size_t)o * Cp + c] = L.w[(size_t)o * Cin + c];
      dycl_status st = dmalloc(g, &L.d_w, wp.size() * 2);
      if (st) return st;
      CK(cudaMemcpy(L.d_w, wp.data(), wp.size() * 2, cudaMemcpyHostToDevice));
      if (L.cout >= 128 && L.cout <= 1024) {
        std::vector<uint16_t> wt((size_t)Cp * L.cout, 0);
        for (int o = 0; o < L.cout; ++o)
          for (int c = 0; c < Cin; ++c) wt[(size_t)c * L.cout + o] = L.w[(size_t)o * Cin + c];
        if ((st = dmalloc(g, &L.d_wt, wt.size() * 2))) return st;
        CK(cudaMemcpy(L.d_wt, wt.data(), wt.size() * 2, cudaMemcpyHostToDevice));
        if (L.out_fp32 && Cp % 32 == 0 && !g->head_cuda_core) {
          // tensor-core head: W2 = [W | W] with N padded to a multiple of 128 (zero rows)
          L.kpad = (L.cout + 127) / 128 * 128;
          std::vector<uint16_t> w2((size_t)L.kpad * 2 * Cp, 0);
          for (int o = 0; o < L.cout; ++o)
            for (int c = 0; c < Cin; ++c) {
              w2[(size_t)o * 2 * Cp + c] = L.w[(size_t)o * Cin + c];
              w2[(size_t)o * 2 * Cp + Cp + c] = L.w[(size_t)o * Cin + c];
            }
          std::vector<float> b2(L.kpad, 0.0f);
          for (int o = 0; o < L.cout && o < (int)L.b.size(); ++o) b2[o] = L.b[o];
          if ((st = dmalloc(g, &L.d_w2, w2.size() * 2))) return st;
          CK(cudaMemcpy(L.d_w2, w2.data(), w2.size() * 2, cudaMemcpyHostToDevice));
          if ((st = dmalloc(g, &L.d_b2, b2.size() * 4))) return st;
          CK(cudaMemcpy(L.d_b2, b2.data(), b2.size() * 4, cudaMemcpyHostToDevice));
        }
      }
    }
    if (!L.b.empty()) {
      dycl_status st = dmalloc(g, &L.d_b, L.b.size() * 4);
      if (st) return st;
      CK(cudaMemcpy(L.d_b, L.b.data(), L.b.size() * 4, cudaMemcpyHostToDevice));
    }
  }
  return DYCL_OK;
}

// ------------------------------------------------------------------ executor
// An activation lives in a bf16 buffer (the tensor-core operand copy) and, for
// residual-stream tensors in DYCL_PREC_FP32_STREAM, also in an fp32 buffer.
struct Tensor {
  int b = -1, f = -1;
};

struct Exec {
  dycl_graph g;
  cudaStream_t st;
  int batch;
  float* out_logits;
  int32_t* out_path;
  float* out_margin = nullptr;       // per-sample min |predicate - threshold| (or nullptr)
  uint16_t* out_features = nullptr;  // dycl_io.features: the final head's input tensor (plain graphs)
  long long global_offset = 0;       // global index of row 0 (rebalanced rows carry their id)
  int own = 0;                       // the rank's own rows (result space rows [0, own))
  int slot = 1;               // next free count slot
  int fused_launch = 0;       // fused-block launches so far in this run (DYCL_TS selection)
  int conv_launch = 0;        // conv launches so far in this run (DYCL_TS_CONV selection)
  int nlaunch = 0;

  void prof_begin(int kind, const int* cnt, double bpr, double fpr, double bfix) {
    if (!g->profiling) return;
    if (g->prof_used >= g->prof.size()) {
      Launch L{};
      cudaEventCreate(&L.e0);
      cudaEventCreate(&L.e1);
      g->prof.push_back(L);
    }
    Launch& L = g->prof[g->prof_used];
    L.kind = kind;
    L.count_dev = cnt;
    L.bytes_per_row = bpr;
    L.flops_per_row = fpr;
    L.bytes_fixed = bfix;
    cudaEventRecord(L.e0, st);
  }
  void prof_end() {
    ++nlaunch;
    if (!g->profiling) return;
    cudaEventRecord(g->prof[g->prof_used].e1, st);
    ++g->prof_used;
  }

  std::vector<dycl::DrbArgs> drb;       // device-rebalanced levels of this run (return path)
  bool pv[dycl_graph_s::NBUF32] = {};   // d_pool32[f] holds the GAP of every live row of buf32[f]
  int gap_f = -1;                       // buf32 index whose GAP sits in d_gap_pooled (conv_gemm fused GAP)
  bool want_gap = false;                // the subnet being run feeds a head: fuse its GAP when possible
  const int* in_rows_gemm = nullptr;    // zero-copy exit into an NHWC bottleneck stage: its first 1x1 conv and
                                        // fused projection read the survivors through this list (no gather)
  const int* in_list = nullptr;         // zero-copy exit: the next subnet's first fused group reads its
                                        // input rows through this list (the survivors) instead of a gather

  Tensor pick_tensor(bool stream, std::initializer_list<Tensor> busy) {
    std::vector<int> bb, bf;
    for (const Tensor& t : busy) {
      bb.push_back(t.b);
      bf.push_back(t.f);
    }
    Tensor o;
    for (int i = 0; i < dycl_graph_s::NBUF && o.b < 0; ++i)
      if (std::find(bb.begin(), bb.end(), i) == bb.end()) o.b = i;
    if (stream)
      for (int i = 0; i < dycl_graph_s::NBUF32 && o.f < 0; ++i)
        if (std::find(bf.begin(), bf.end(), i) == bf.end()) o.f = i;
    if (o.f >= 0) pv[o.f] = false;               // about to be rewritten
    if (o.f >= 0 && o.f == gap_f) gap_f = -1;
    return o;
  }
  bool fp32_stream() const { return g->precision == DYCL_PREC_FP32_STREAM; }
  // bf16 activation layout of a tensor with C (padded) channels: NHWC when C % 64 == 0 (the
  // im2col GEMM's 64-channel operand boxes), channel-planar otherwise (the two coincide at C = 8)
  bool lay(int C) const { return g->nhwc && C % 64 == 0; }

  // A basic block the fused kernel can run: BLOCK, conv3x3/s1/p1 ReLU (C->C),
  // conv3x3/s1/p1 ReLU + identity residual, on an eligible sample shape.
  static bool fusable(const Subnet& s, size_t li) {
    if (li + 2 >= s.layers.size()) return false;
    const Layer &B = s.layers[li], &c1 = s.layers[li + 1], &c2 = s.layers[li + 2];
    if (B.kind != L_BLOCK || c1.kind != L_CONV || c2.kind != L_CONV) return false;
    for (const Layer* c : {&c1, &c2})
      if (c->k != 3 || c->stride != 1 || c->pad != 1 || !c->relu || !c->d_wrt || c->in.C != c->out.C ||
          !(c->in == c->out))
        return false;
    if (c1.residual || !c2.residual || c2.res_mode != 1) return false;
    return dycl::block_fused_eligible(c1.in.C, c1.in.H, c1.in.W);
  }

  // A gate then-branch [block, 3x3/1/1 conv + ReLU, 3x3/1/1 conv + identity shortcut + ReLU] on
  // NHWC tensors whose samples tile 128-row GEMM tiles whole: the in-place GEMM form applies.
  bool inplace_gemm_ok(const Subnet& T) const {
    if (T.layers.size() != 3 || T.layers[0].kind != L_BLOCK) return false;
    const Layer &c1 = T.layers[1], &c2 = T.layers[2];
    for (const Layer* c : {&c1, &c2})
      if (c->kind != L_CONV || c->k != 3 || c->stride != 1 || c->pad != 1 || !c->relu || !(c->in == c->out) ||
          c->fuse_proj || c->s4d || c->s2d2)
        return false;
    const int hw = c1.in.H * c1.in.W;
    return !c1.residual && c2.residual && c2.res_mode == 1 && lay(c1.in.Cp()) && lay(c1.out.C) && hw <= 128 &&
           128 % hw == 0 && hw % 8 == 0;
  }

  // A sub-network the NHWC GEMM can enter zero-copy: [block, 1x1/s1 conv, ..., projection fused
  // into the block's last conv] whose samples split into row-list boxes (dycl::zero_copy_rows:
  // 56x56 -> 64-row A / 16-pixel projection boxes; 28x28 -> 16 / 4, 14x14 -> 4 / 1) -- the block
  // input is read only by the first conv and by the projection, both through the row list.
  // Projection boxes below zc_proj_min pixels (default 8) are not used: at 28x28 the 4-pixel
  // boxes (32 TMA requests per k-block) slow the stage's first conv3 + projection GEMM by more
  // than the gather they save (cfg 5: 931 -> 944 ms per step; DYCL_ZC_PROJ_MIN=4 enables them).
  bool gemm_list_entry(const Subnet& S) const {
    if (S.layers.size() < 5 || S.layers[0].kind != L_BLOCK) return false;
    const Layer& c1 = S.layers[1];
    if (c1.kind != L_CONV || c1.k != 1 || c1.stride != 1 || c1.residual || c1.s4d || c1.s2d2 || !lay(c1.in.Cp()) ||
        !lay(c1.out.C) || dycl::zero_copy_rows(c1.in.H * c1.in.W, 64) < dycl::ZC_MIN_ROWS || c1.in.Cp() % 64 ||
        c1.out.C % 64)
      return false;
    for (size_t li = 2; li < S.layers.size() && S.layers[li].kind != L_BLOCK; ++li) {
      const Layer& L = S.layers[li];
      if (L.kind == L_PROJ)
        return li + 1 < S.layers.size() && S.layers[li + 1].fuse_proj &&
               dycl::zero_copy_rows(S.layers[li + 1].out.H * S.layers[li + 1].out.W, 16) >= g->zc_proj_min;
      if (L.residual) return false;
    }
    return false;
  }

  // Run subnet s on the rows of `in` (device count `cnt`).  The last layer writes
  // into `out_hint` when given (b >= 0).  `busy` is an outer tensor to preserve.
  dycl_status subnet(const Subnet& s, Tensor in, const int* cnt, Tensor out_hint, Tensor busy, Tensor* out) {
    Tensor cur = in, shortcut, proj_src;
    for (size_t li = 0; li < s.layers.size(); ++li) {
      const Layer& L = s.layers[li];
      if (in_list && !(li == 0 && L.kind == L_BLOCK && fp32_stream() && !g->no_fuse && cur.f >= 0 && fusable(s, li)))
        return fail(g, DYCL_E_STATE, "internal: zero-copy input on a non-fused first layer");
      if (L.kind == L_BLOCK && fp32_stream() && !g->no_fuse && cur.f >= 0 && fusable(s, li)) {
        // up to MAX_FUSED_BLOCKS consecutive fusable blocks (same shape) in one launch
        int nb = 1;
        while (nb < dycl::MAX_FUSED_BLOCKS && nb < g->max_fuse && fusable(s, li + 3 * nb) &&
               s.layers[li + 3 * nb + 1].in == s.layers[li + 1].in)
          ++nb;
        const Layer &c1 = s.layers[li + 1], &c2 = s.layers[li + 2];
        const size_t lend = li + 3 * nb;             // first layer after the fused group
        const bool last = lend == s.layers.size();
        const bool need_b = last || !fusable(s, lend);   // the next layer reads the bf16 copy
        Tensor o = (last && out_hint.b >= 0) ? out_hint : pick_tensor(true, {cur, busy, out_hint});
        if (o.b < 0 || o.f < 0) return fail(g, DYCL_E_STATE, "internal: out of activation buffers");
        dycl::BlockArgs ba{};
        ba.x32 = g->buf32[cur.f];
        ba.y32 = g->buf32[o.f];
        ba.yb = need_b ? g->buf[o.b] : nullptr;
        ba.nblk = nb;
        ba.list = in_list;                           // input rows = survivors of the last exit (zero-copy)
        in_list = nullptr;
        for (int k = 0; k < nb; ++k) {
          ba.w1_rt[k] = s.layers[li + 3 * k + 1].d_wrt;
          ba.w2_rt[k] = s.layers[li + 3 * k + 2].d_wrt;
          ba.b1[k] = s.layers[li + 3 * k + 1].d_b;
          ba.b2[k] = s.layers[li + 3 * k + 2].d_b;
        }
        ba.n_live = cnt;
        ba.C = c1.in.C; ba.H = c1.in.H; ba.W = c1.in.W;
        ba.pooled = last ? g->d_pool32[o.f] : nullptr;   // fused GAP for the head that follows the subnet
        ++fused_launch;
        ba.ts = (g->dbg_ts_pick == 0 || g->dbg_ts_pick == fused_launch) ? g->dbg_ts : nullptr;
        const double row_b = (4.0 + 4.0 + (need_b ? 2.0 : 0.0)) * c1.in.row_elems();
        const double row_f = nb * 2.0 * 2.0 * c1.out.H * c1.out.W * c1.out.C * (double)(9 * c1.in.C);
        prof_begin(DYCL_K_BLOCK, cnt, row_b, row_f, nb * 2.0 * 2 * 3 * c1.out.C * c1.Kp_rt);
        cudaError_t e = dycl::launch_block_fused(ba, batch, g->num_sms, st);
        prof_end();
        if (e != cudaSuccess) return cuda_fail(g, e, "launch_block_fused");
        if (!need_b) o.b = -1;                        // no valid bf16 copy
        pv[o.f] = ba.pooled != nullptr;
        cur = o;
        li = lend - 1;
        continue;
      }
      if (L.kind == L_BLOCK) {
        shortcut = cur;
        continue;
      }
      if (L.kind == L_GAP || (L.kind == L_DENSE && L.out_fp32))
        return fail(g, DYCL_E_UNSUPPORTED, "head layers inside a sequential subnet");
      const bool last = li + 1 == s.layers.size();
      if (L.kind == L_MAXPOOL) {
        // the pool output is a residual-stream tensor only if something reads its fp32 copy: a
        // block whose shortcut is a projection reads its input as the bf16 operand alone
        bool proj_next = false;
        if (!last && s.layers[li + 1].kind == L_BLOCK)
          for (size_t lj = li + 2; lj < s.layers.size() && s.layers[lj].kind != L_BLOCK; ++lj)
            proj_next = proj_next || s.layers[lj].kind == L_PROJ;
        const bool stream_mp = fp32_stream() && (last || s.layers[li + 1].kind == L_BLOCK) && !proj_next;
        Tensor o = (last && out_hint.b >= 0) ? out_hint : pick_tensor(stream_mp, {cur, shortcut, busy, out_hint});
        if (o.b < 0 || (stream_mp && o.f < 0)) return fail(g, DYCL_E_STATE, "internal: out of activation buffers");
        if (!stream_mp) o.f = -1;
        dycl::PoolArgs pa{};
        pa.x = g->buf[cur.b];
        pa.x32 = cur.f >= 0 ? g->buf32[cur.f] : nullptr;
        pa.y = g->buf[o.b];
        pa.y32 = o.f >= 0 ? g->buf32[o.f] : nullptr;
        pa.n_live = cnt;
        pa.H = L.in.H; pa.W = L.in.W; pa.C = L.in.Cp(); pa.Ho = L.out.H; pa.Wo = L.out.W;
        pa.k = L.k; pa.stride = L.stride; pa.pad = L.pad;
        pa.nhwc = lay(L.in.Cp());
        pa.s2d = L.pool_s2d;
        prof_begin(DYCL_K_POOL, cnt, (pa.x32 ? 4.0 : 2.0) * L.in.row_elems() + (o.f >= 0 ? 6.0 : 2.0) * L.out.row_elems(), 0, 0);
        cudaError_t e = dycl::launch_maxpool(pa, batch, g->num_sms, st);
        prof_end();
        if (e != cudaSuccess) return cuda_fail(g, e, "launch_maxpool");
        cur = o;
        continue;
      }
      if (L.kind == L_PROJ && li + 1 < s.layers.size() && s.layers[li + 1].fuse_proj) {
        proj_src = shortcut;           // consumed by the next conv's fused GEMM
        continue;
      }
      if (L.kind == L_PROJ) {
        // shortcut <- conv1x1/stride(shortcut): a residual-stream tensor
        Tensor o = pick_tensor(fp32_stream(), {cur, shortcut, busy, out_hint});
        if (o.b < 0 || (fp32_stream() && o.f < 0)) return fail(g, DYCL_E_STATE, "internal: out of activation buffers");
        if (!fp32_stream()) o.f = -1;
        dycl::ConvArgs a{};
        a.x = g->buf[shortcut.b];
        a.w = L.d_w;
        a.bias = L.d_b;
        a.y = g->buf[o.b];
        a.y32 = o.f >= 0 ? g->buf32[o.f] : nullptr;
        a.n_live = cnt;
        a.H = L.in.H; a.W = L.in.W; a.C = L.in.Cp();
        a.Ho = L.out.H; a.Wo = L.out.W; a.Cout = L.out.C;
        a.ksz = 1; a.stride = L.stride; a.pad = 0;
        a.K = L.K; a.Kp = L.Kp;
        a.relu = 0;
        a.in_nhwc = lay(L.in.Cp());
        a.nhwc = lay(L.out.C);
        a.dbg = g->conv_dbg;
        a.y32_pair = g->stream_pair;
        prof_begin(DYCL_K_CONV, cnt, 2.0 * L.in.row_elems() + (o.f >= 0 ? (g->stream_pair ? 4.0 : 6.0) : 2.0) * L.out.row_elems(),
                   2.0 * L.out.H * L.out.W * L.out.C * (double)L.in.C, 2.0 * L.out.C * L.Kp);
        cudaError_t e = dycl::launch_conv(a, batch, g->num_sms, st, g->conv_path);
        prof_end();
        if (e != cudaSuccess) return cuda_fail(g, e, "launch_conv(projection)");
        shortcut = o;
        continue;
      }
      const bool stream = fp32_stream() && (last || L.residual || s.layers[li + 1].kind == L_BLOCK);
      Tensor o = (last && out_hint.b >= 0) ? out_hint : pick_tensor(stream, {cur, shortcut, busy, out_hint});
      if (o.b < 0 || (stream && o.f < 0)) return fail(g, DYCL_E_STATE, "internal: out of activation buffers");
      if (!stream) o.f = -1;
      dycl::ConvArgs a{};
      a.x = g->buf[cur.b];
      a.w = L.d_w;
      a.w_rt = L.d_wrt;
      a.Kp_rt = L.Kp_rt;
      a.bias = L.d_b;
      a.res = L.res_mode ? g->buf[shortcut.b] : nullptr;
      a.res32 = (L.res_mode && shortcut.f >= 0) ? g->buf32[shortcut.f] : nullptr;
      a.y = g->buf[o.b];
      a.y32 = o.f >= 0 ? g->buf32[o.f] : nullptr;
      a.n_live = cnt;
      a.n_static = 0;
      a.H = L.in.H; a.W = L.in.W; a.C = L.in.Cp();
      a.Ho = L.out.H; a.Wo = L.out.W; a.Cout = L.out.C;
      a.ksz = L.k; a.stride = L.stride; a.pad = L.pad;
      a.K = L.K; a.Kp = L.Kp;
      a.relu = L.relu;
      a.res_mode = L.res_mode;
      a.rH = L.res_shape.H; a.rW = L.res_shape.W; a.rC = L.res_shape.Cp();
      a.r_pad_lo = (L.out.C - L.res_shape.C) / 2;
      a.in_nhwc = lay(L.in.Cp());
      a.nhwc = lay(L.out.C);
      a.res_nhwc = lay(L.res_shape.Cp());
      double fused_b = 0.0, fused_f = 0.0;
      if (L.fuse_proj) {               // [t | x] x [W | W_proj]: no projection tensor, no shortcut read
        const Layer& Pj = s.layers[li - 1];
        a.x2 = g->buf[proj_src.b];
        a.C2 = Pj.in.C; a.H2 = Pj.in.H; a.W2 = Pj.in.W; a.stride2 = Pj.stride;
        a.K = a.Kp = L.in.C + Pj.in.C;
        a.w = L.d_wcat;
        a.bias = L.d_bcat;
        a.res_mode = 0;
        a.res = nullptr;
        a.res32 = nullptr;
        fused_b = 2.0 * L.out.H * L.out.W * Pj.in.C;   // the strided pixels of x the GEMM reads
        fused_f = 2.0 * L.out.H * L.out.W * L.out.C * (double)Pj.in.C;
      }
      if (L.s2d2) {                    // 4x4 / stride 1 over 2x2 blocks (pad 2 before, 1 after)
        a.H = L.in.H / 2; a.W = L.in.W / 2; a.C = 16;
        a.Ho = L.out.H; a.Wo = L.out.W; a.Cout = L.out.C;
        a.ksz = 4; a.stride = 1; a.pad = 2;
        a.K = a.Kp = 16 * 16;
        a.w_rt = nullptr;
        a.in_nhwc = a.nhwc = 1;
      }
      if (L.s4d) {                     // 3x3 / stride 1 over 4x4 blocks, 2x2 output phases in N
        a.H = L.in.H / 4; a.W = L.in.W / 4; a.C = 64;
        a.Ho = L.out.H / 2; a.Wo = L.out.W / 2; a.Cout = 4 * L.out.C;
        a.ksz = 3; a.stride = 1; a.pad = 1;
        a.K = a.Kp = 9 * 64;
        a.c_live = g->halo_kskip ? 16 * L.in.C : 0;   // 4x4 pixels x C real channels per block; the rest zero
        a.w_rt = nullptr;
        a.in_nhwc = a.nhwc = 1;
      }
      // the fused block group that follows reads only the fp32 stream: skip the bf16 copy
      const bool skip_b = !last && o.f >= 0 && fp32_stream() && !g->no_fuse && !L.s4d &&
                          s.layers[li + 1].kind == L_BLOCK && fusable(s, li + 1);
      if (skip_b) a.y = nullptr;
      a.dbg = g->conv_dbg;
      a.y32_pair = g->stream_pair;
      if (in_rows_gemm && li == 1) a.rows_gather = in_rows_gemm;     // zero-copy entry (gemm_list_entry)
      if (in_rows_gemm && L.fuse_proj) {
        a.x2_rows = in_rows_gemm;
        in_rows_gemm = nullptr;                      // the block input has no other reader
      }
      const double res_b = a.res_mode ? (a.res32 ? 4.0 : 2.0) * L.res_shape.row_elems() *
                                            (a.res_mode == 2 ? 0.25 : 1.0) : 0.0;
      const double row_b = 2.0 * L.in.row_elems() +
                           (o.f >= 0 ? (a.y ? 2.0 : 0.0) + (g->stream_pair ? 2.0 : 4.0) : 2.0) * L.out.row_elems() + res_b +
                           fused_b;
      const double row_f = 2.0 * L.out.H * L.out.W * L.out.C * (double)(L.k * L.k * L.in.C) + fused_f;
      // (only for wide rows: below ~128 KB of fp32 per sample the head's own GAP pass is cheaper)
      const bool gap = want_gap && last && g->d_gap_part && a.y32 && a.nhwc && a.in_nhwc && !a.rows_out &&
                       gap_group(L.out.H * L.out.W) >= 4 &&
                       L.out.H * L.out.W >= 32 && 4.0 * L.out.row_elems() >= 128 * 1024 &&
                       dycl::conv_gemm_eligible(a);
      const int gap_g = gap_group(L.out.H * L.out.W);
      if (gap) {
        a.gap_part = g->d_gap_part;
        a.gap_g = gap_g;
      }
      ++conv_launch;
      if (g->dbg_ts_conv && g->dbg_ts_conv == conv_launch) a.ts = g->dbg_ts;
      prof_begin(DYCL_K_CONV, cnt, row_b, row_f, 2.0 * L.out.C * L.Kp);
      cudaError_t e = dycl::launch_conv(a, batch, g->num_sms, st, g->conv_path);
      prof_end();
      if (e != cudaSuccess) return cuda_fail(g, e, "launch_conv_tc");
      if (gap) {
        prof_begin(DYCL_K_HEAD, cnt, 4.0 * (L.out.H * L.out.W / gap_g) * L.out.C + 4.0 * L.out.C, 0, 0);
        e = dycl::launch_gap_reduce(g->d_gap_part, gap_g, g->d_gap_pooled, cnt, batch, L.out.H * L.out.W, L.out.C, st);
        prof_end();
        if (e != cudaSuccess) return cuda_fail(g, e, "launch_gap_reduce");
        gap_f = o.f;
      }
      if (!a.y) o.b = -1;                            // only the fp32 copy was written
      cur = o;
    }
    *out = cur;
    return DYCL_OK;
  }

  dycl_status head(const Subnet& s, Tensor in, const int* cnt, int kind, float thr) {
    const Layer& D = s.layers.back();
    dycl::HeadArgs a{};
    a.h = in.b >= 0 ? g->buf[in.b] : nullptr;
    a.h32 = in.f >= 0 ? g->buf32[in.f] : nullptr;
    a.h32_pair = g->stream_pair;
    if (a.h32_pair && a.h32 && !a.h) return fail(g, DYCL_E_STATE, "internal: pair stream head without its hi plane");
    a.w = D.d_w;
    a.b = D.d_b;
    a.z = g->d_z;
    a.flag = g->d_flag;
    a.pred = g->d_pred;
    a.n_live = cnt;
    a.HW = s.in.H * s.in.W;
    a.C = s.in.Cp();
    a.K = D.cout;
    a.kind = kind;
    a.thr = thr;
    a.nhwc = lay(s.in.Cp());
    if (in.f >= 0 && g->d_pool32[in.f] && s.in.H * s.in.W > 1 && s.in.Cp() <= 32) {
      if (pv[in.f]) a.pooled = g->d_pool32[in.f];
      else a.pooled_out = g->d_pool32[in.f];     // computed here, kept for the in-place gates that follow
    }
    if (D.d_wt && kind != 1 && g->d_gpool) {
      a.wt = D.d_wt;
      a.gpool = g->d_gpool;
      if (D.d_w2 && g->d_a2) {
        a.w2 = D.d_w2;
        a.b2 = D.d_b2;
        a.a2 = g->d_a2;
        a.kpad = D.kpad;
      }
    }
    a.num_sms = g->num_sms;
    if (in.f >= 0 && in.f == gap_f && g->d_gap_pooled) a.pooled = g->d_gap_pooled;   // GAP fused into the producer
    prof_begin(DYCL_K_HEAD, cnt, (a.h32 ? 4.0 : 2.0) * s.in.row_elems() + 4.0 * D.cout + 1,
               2.0 * D.cout * s.in.C + s.in.row_elems(), 2.0 * D.cout * a.C);
    cudaError_t e = dycl::launch_head(a, batch, st);
    prof_end();
    if (e != cudaSuccess) return cuda_fail(g, e, "launch_head");
    if (a.pooled_out) pv[in.f] = true;
    return DYCL_OK;
  }

  dycl_status compact(const int* cnt, int mode, int32_t bit, int orig_cur, int* s_out, bool pred, float thr) {
    *s_out = slot;
    if (slot + 2 > g->n_slots) return fail(g, DYCL_E_STATE, "count slots exhausted");
    prof_begin(DYCL_K_COMPACT, cnt, 1.0 + 4 * 4 + (pred && out_margin ? 12.0 : 0.0), 0, 0);
    cudaError_t e = dycl::launch_compact(g->d_flag, cnt, g->d_orig[orig_cur], g->d_list1, g->d_list0,
                                         g->d_counts + slot, g->d_orig[orig_cur ^ 1], mode, out_path, bit,
                                         g->d_pred, thr, pred ? out_margin : nullptr, st);
    prof_end();
    slot += 2;
    if (e != cudaSuccess) return cuda_fail(g, e, "launch_compact");
    return DYCL_OK;
  }

  dycl_status scatter(const int* list, const int* count, int orig_cur, int32_t path_val) {
    prof_begin(DYCL_K_SCATTER, count, 2.0 * 4 * g->K + 12, 0, 0);
    cudaError_t e = dycl::launch_scatter(g->d_z, g->K, list, count, g->d_orig[orig_cur], out_logits, out_path,
                                         path_val, batch, st);
    prof_end();
    if (e != cudaSuccess) return cuda_fail(g, e, "launch_scatter");
    return DYCL_OK;
  }

  // Copy rows list[j] of `src` into rows (*off + j) of `dst` (identity or option A),
  // for each precision copy the source tensor carries.
  dycl_status gather(Tensor src, Tensor dst, const int* list, const int* count, const int* off, const Shape& sh,
                     int mode) {
    for (int pass = 0; pass < 2; ++pass) {
      const int si = pass == 0 ? src.b : src.f, di = pass == 0 ? dst.b : dst.f;
      if (si < 0) continue;
      if (di < 0) return fail(g, DYCL_E_STATE, "internal: gather destination lacks a copy");
      dycl::GatherArgs a{};
      a.elem_bytes = pass == 0 || g->stream_pair ? 2 : 4;
      a.src = pass == 0 ? (const void*)g->buf[si] : (const void*)g->buf32[si];
      a.dst = pass == 0 ? (void*)g->buf[di] : (void*)g->buf32[di];
      a.list = list;
      a.count = count;
      a.dst_off_count = off;
      a.row_elems_src = sh.row_elems();
      a.mode = mode;
      a.H = sh.H; a.W = sh.W; a.C = sh.Cp();
      a.row_elems_dst = mode == 0 ? sh.row_elems() : (long long)(sh.H / 2) * (sh.W / 2) * 2 * sh.Cp();
      a.dst_nhwc = mode == 1 && lay(2 * sh.Cp());
      const double eb = a.elem_bytes;
      prof_begin(DYCL_K_GATHER, count, eb * (mode == 0 ? a.row_elems_src : a.row_elems_dst / 2) + eb * a.row_elems_dst,
                 0, 0);
      cudaError_t e = dycl::launch_gather(a, batch, g->num_sms, st);
      prof_end();
      if (e != cudaSuccess) return cuda_fail(g, e, "launch_gather");
    }
    return DYCL_OK;
  }

  dycl_status run(const float* input) {
    dycl_status r;
    int orig_cur = 0;
    prof_begin(DYCL_K_INIT, nullptr, 0, 0, 12.0 * batch);
    cudaError_t e = dycl::launch_init(g->d_counts, own, g->d_orig[0], out_path, out_margin, batch, st);
    prof_end();
    if (e != cudaSuccess) return cuda_fail(g, e, "launch_init");
    if (g->tr && g->rb_device && g->rb_policy != 0 && g->n_exits > 0) {
      e = dycl::drb_begin(g->d_drb_epoch, st);           // this run's exchange epoch (every rank)
      if (e != cudaSuccess) return cuda_fail(g, e, "drb_begin");
    }
    if (g->d_rnn_state) {
      e = cudaMemsetAsync(g->d_rnn_state, 0, (size_t)batch * 2 * g->rnn_hidden * sizeof(float), st);
      if (e != cudaSuccess) return cuda_fail(g, e, "rnn state reset");
    }
    const Shape& in = g->input;
    prof_begin(DYCL_K_INPUT, nullptr, 0, 0, (double)batch * in.H * in.W * (4.0 * in.C + 2.0 * in.Cp()));
    e = own == 0 ? cudaSuccess
        : g->stem_s2d2 ? dycl::launch_cast_s2d2(input, g->buf[0], own, in.H, in.W, in.C, st)
        : g->stem_s4d ? dycl::launch_cast_s4d(input, g->buf[0], own, in.H, in.W, in.C, st)
                      : dycl::launch_cast_pad(input, g->buf[0], own, in.H * in.W, in.C, in.Cp(), st);
    prof_end();
    if (e != cudaSuccess) return cuda_fail(g, e, "launch_cast_pad");
    Tensor cur;
    cur.b = 0;
    const int* cnt = g->d_counts;
    const Tensor none;
    for (size_t ni = 0; ni < g->nodes.size(); ++ni) {
      const Node& N = g->nodes[ni];
      switch (N.kind) {
        case N_SEQ: {
          Tensor o;
          want_gap = ni + 1 < g->nodes.size() &&
                     (g->nodes[ni + 1].kind == N_EXIT || g->nodes[ni + 1].kind == N_FINAL);
          r = subnet(g->subnets[N.sn], cur, cnt, none, none, &o);
          want_gap = false;
          if (r) return r;
          cur = o;
          break;
        }
        case N_EXIT: {
          if ((r = head(g->subnets[N.sn], cur, cnt, 0, N.thr))) return r;
          int s;
          if ((r = compact(cnt, 0, 0, orig_cur, &s, true, N.thr))) return r;
          if ((r = scatter(g->d_list1, g->d_counts + s, orig_cur, N.ordinal))) return r;
          const bool rebal = rebalance_here(N.ordinal);
          // survivors move on; their fp32 stream copy only if the next reader uses it (a
          // ResNet-50 stage starts with a projection block: its input is read as bf16 only)
          const bool next_seq = ni + 1 < g->nodes.size() && g->nodes[ni + 1].kind == N_SEQ;
          const bool keep32 = cur.f >= 0 && !(next_seq && !g->subnets[g->nodes[ni + 1].sn].needs_in32);
          // ... and their bf16 copy only if the next reader is not a fused block (which reads the
          // fp32 stream alone).  A fused block can even read the survivors in place through the
          // compaction's row list: then nothing moves at all (zero-copy exit)
          const bool next_fused = next_seq && keep32 && fp32_stream() && !g->no_fuse &&
                                  fusable(g->subnets[g->nodes[ni + 1].sn], 0);
          if (next_fused && !g->no_zero_copy && !rebal) {
            in_list = g->d_list0;
            cnt = g->d_counts + s + 1;
            orig_cur ^= 1;
            break;
          }
          if (next_seq && !g->no_zero_copy && !rebal && gemm_list_entry(g->subnets[g->nodes[ni + 1].sn])) {
            in_rows_gemm = g->d_list0;                 // the next stage reads the survivors in place
            cnt = g->d_counts + s + 1;
            orig_cur ^= 1;
            break;
          }
          const bool keepb = !next_fused;
          Tensor src = cur;
          if (!keep32) src.f = -1;
          if (!keepb) src.b = -1;
          Tensor nb = pick_tensor(keep32, {cur});
          if (!keep32) nb.f = -1;
          if (!keepb) nb.b = -1;
          if ((r = gather(src, nb, g->d_list0, g->d_counts + s + 1, nullptr, N.in, 0))) return r;
          cur = nb;
          cnt = g->d_counts + s + 1;
          orig_cur ^= 1;
          if (rebal && (r = rebalance(cur, g->d_counts + s + 1, N.in, orig_cur))) return r;
          break;
        }
        case N_GATE: {
          if (N.rnn) {
            // u = proj(h) into d_z (no predicate), then the shared LSTM cell steps on u for every
            // live row (state indexed by the row's original sample), z = w_out . h, sigmoid > thr
            if ((r = head(g->subnets[N.sn], cur, cnt, 2, 0.f))) return r;
            dycl::RnnGateArgs ra{};
            ra.u = g->d_z;
            ra.u_stride = std::max(g->K, 1);
            ra.orig = g->d_orig[orig_cur];
            ra.state = g->d_rnn_state;
            ra.w = g->d_rnn_w;
            ra.w_out = N.d_w_out;
            ra.b_out = N.b_out;
            ra.n_in = g->rnn_in;
            ra.hidden = g->rnn_hidden;
            ra.thr = N.thr;
            ra.flag = g->d_flag;
            ra.pred = g->d_pred;
            ra.n_live = cnt;
            const double H4 = 4.0 * g->rnn_hidden;
            prof_begin(DYCL_K_HEAD, cnt, 4.0 * g->rnn_in + 2 * 8.0 * g->rnn_hidden + 5.0,
                       2.0 * H4 * (g->rnn_in + g->rnn_hidden) + 2.0 * g->rnn_hidden, 0);
            cudaError_t e = dycl::launch_rnn_gate(ra, batch, g->num_sms, st);
            prof_end();
            if (e != cudaSuccess) return cuda_fail(g, e, "launch_rnn_gate");
          } else if ((r = head(g->subnets[N.sn], cur, cnt, 1, N.thr))) {
            return r;
          }
          int s;
          if ((r = compact(cnt, 1, (int32_t)1 << N.ordinal, orig_cur, &s, true, N.thr))) return r;
          const Subnet& T = g->subnets[N.then_sn];
          if (N.skip_mode == 0 && fp32_stream() && cur.f >= 0 && cur.b >= 0 && !g->no_fuse && !g->no_inplace &&
              T.layers.size() == 3 && fusable(T, 0)) {
            // in place (the slot-table form of the skip, P:L648 identity elimination): the
            // executed rows' block output overwrites their own rows, skipped rows are not
            // touched -- no gather, no merge, row order and orig unchanged
            const Layer &c1 = T.layers[1], &c2 = T.layers[2];
            dycl::BlockArgs ba{};
            ba.x32 = g->buf32[cur.f];
            ba.y32 = g->buf32[cur.f];
            ba.yb = g->buf[cur.b];
            ba.list = g->d_list1;
            ba.list_out = 1;
            ba.nblk = 1;
            ba.w1_rt[0] = c1.d_wrt;
            ba.w2_rt[0] = c2.d_wrt;
            ba.b1[0] = c1.d_b;
            ba.b2[0] = c2.d_b;
            ba.n_live = g->d_counts + s;
            ba.C = c1.in.C; ba.H = c1.in.H; ba.W = c1.in.W;
            ba.ts = nullptr;
            ba.pooled = pv[cur.f] ? g->d_pool32[cur.f] : nullptr;   // executed rows refresh their GAP
            const double row_b = (4.0 + 4.0 + 2.0) * c1.in.row_elems();
            const double row_f = 2.0 * 2.0 * c1.out.H * c1.out.W * c1.out.C * (double)(9 * c1.in.C);
            prof_begin(DYCL_K_BLOCK, g->d_counts + s, row_b, row_f, 2.0 * 2 * 3 * c1.out.C * c1.Kp_rt);
            cudaError_t e = dycl::launch_block_fused(ba, batch, g->num_sms, st);
            prof_end();
            if (e != cudaSuccess) return cuda_fail(g, e, "launch_block_fused (in place)");
            if (gap_f == cur.f) gap_f = -1;
            break;
          }
          if (N.skip_mode == 0 && !g->no_inplace && cur.b >= 0 && inplace_gemm_ok(T)) {
            // in place on the NHWC GEMM (whole-sample tiles): conv1 reads the executed rows
            // through the list into a dense scratch T, conv2 writes y (+ the fp32 stream) back
            // over those rows, its identity shortcut read from the same rows
            const Layer &c1 = T.layers[1], &c2 = T.layers[2];
            const int* ecnt = g->d_counts + s;
            const Tensor tt = pick_tensor(false, {cur});
            if (tt.b < 0) return fail(g, DYCL_E_STATE, "internal: out of activation buffers");
            for (int k = 0; k < 2; ++k) {
              const Layer& L = k == 0 ? c1 : c2;
              dycl::ConvArgs a{};
              a.x = k == 0 ? g->buf[cur.b] : g->buf[tt.b];
              a.w = L.d_w;
              a.w_rt = L.d_wrt;
              a.Kp_rt = L.Kp_rt;
              a.bias = L.d_b;
              a.n_live = ecnt;
              a.H = L.in.H; a.W = L.in.W; a.C = L.in.Cp();
              a.Ho = L.out.H; a.Wo = L.out.W; a.Cout = L.out.C;
              a.ksz = L.k; a.stride = L.stride; a.pad = L.pad;
              a.K = L.K; a.Kp = L.Kp;
              a.relu = L.relu;
              a.in_nhwc = a.nhwc = 1;
              if (k == 0) {
                a.rows_in = g->d_list1;
                a.y = g->buf[tt.b];
              } else {
                a.rows_out = g->d_list1;
                a.y = g->buf[cur.b];
                a.y32 = cur.f >= 0 ? g->buf32[cur.f] : nullptr;
                a.res_mode = 1;
                a.res32 = cur.f >= 0 ? g->buf32[cur.f] : nullptr;
                a.res = g->buf[cur.b];
                a.rH = L.out.H; a.rW = L.out.W; a.rC = L.out.C;
              }
              a.dbg = g->conv_dbg;
              const double row_b = 2.0 * L.in.row_elems() + (k == 1 && cur.f >= 0 ? 10.0 : 2.0) * L.out.row_elems();
              const double row_f = 2.0 * L.out.H * L.out.W * L.out.C * (double)(L.k * L.k * L.in.C);
              prof_begin(DYCL_K_CONV, ecnt, row_b, row_f, 2.0 * L.out.C * L.Kp);
              cudaError_t e = dycl::launch_conv(a, batch, g->num_sms, st, g->conv_path);
              prof_end();
              if (e != cudaSuccess) return cuda_fail(g, e, "launch_conv (in place)");
            }
            if (cur.f >= 0) pv[cur.f] = false;
            if (gap_f == cur.f) gap_f = -1;
            break;
          }
          Tensor bt = pick_tensor(false, {cur});
          bt.f = -1;
          Tensor in_t = cur;
          in_t.f = -1;   // the then-branch reads only the bf16 operand copy ...
          if ((r = gather(in_t, bt, g->d_list1, g->d_counts + s, nullptr, N.in, 0))) return r;
          // ... except its shortcut: give the branch the fp32 rows too when streaming
          if (cur.f >= 0) {
            const Tensor bt32 = pick_tensor(true, {cur, bt});
            bt.f = bt32.f;
            Tensor src = cur;
            src.b = -1;
            Tensor dst = bt;
            dst.b = -1;
            if ((r = gather(src, dst, g->d_list1, g->d_counts + s, nullptr, N.in, 0))) return r;
          }
          const bool stream = fp32_stream();
          const Tensor merged = pick_tensor(stream, {cur, bt});
          Tensor o;
          if ((r = subnet(g->subnets[N.then_sn], bt, g->d_counts + s, merged, cur, &o))) return r;
          if ((r = gather(cur, merged, g->d_list0, g->d_counts + s + 1, g->d_counts + s, N.in, N.skip_mode))) return r;
          if (merged.f >= 0) pv[merged.f] = false;   // the skipped rows just arrived without a pooled copy
          cur = merged;
          if (!stream) cur.f = -1;
          orig_cur ^= 1;
          break;
        }
        case N_FINAL: {
          if (out_features) {
            // the encoder output of an En-Decoder: rows are in input order in a plain graph
            if (g->n_exits || g->n_gates || cur.b < 0 || !lay(N.in.Cp()) || N.in.C % 64)
              return fail(g, DYCL_E_UNSUPPORTED, "features output: plain graphs with an NHWC final tensor only");
            e = cudaMemcpyAsync(out_features, g->buf[cur.b], (size_t)batch * N.in.row_elems() * 2,
                                cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) return cuda_fail(g, e, "features copy");
          }
          if ((r = head(g->subnets[N.sn], cur, cnt, 2, 0.f))) return r;
          int s;
          if ((r = compact(cnt, 0, 0, orig_cur, &s, false, 0.f))) return r;
          const int32_t pv = g->n_exits > 0 ? g->n_exits : -1;
          if ((r = scatter(g->d_list1, g->d_counts + s, orig_cur, pv))) return r;
          break;
        }
      }
    }
    return return_results();
  }

  // ---------------------------------------------------------------- a9 rebalancing
  struct Level {
    std::vector<int> send, recv;     // rows to / from each rank
    int ext0 = 0;                    // result-space id of the first row received at this level
    long long sent0 = 0;             // offset of this level's rows in d_sent_orig / d_ret_*
    int n_send = 0, n_recv = 0;
    bool moved_any = false;          // some rank moved rows at this level (all ranks agree)
  };
  std::vector<Level> levels;
  int ext_used = 0;
  long long sent_used = 0;

  bool rebalance_here(int exit_ordinal) const {
    return g->tr && !g->rnn_hidden && exit_ordinal < 31 && (g->rb_policy >> exit_ordinal) & 1;
  }

  // After an exit: the survivors sit dense in rows [0, s) of t.  All ranks agree on the counts
  // (all-gather), compute the same deterministic plan (dycl_rebalance_plan), and exchange the
  // surplus rows -- the LAST rows of a surplus rank, in order -- with their metadata; arrivals
  // are appended after the local survivors and get result-space ids past the own rows.
  // Device-initiated form: counts, plan, row transfer and bookkeeping all on the
  // device (drb.cu); level k's received rows get result ids [max_batch * (1 + k), ...), its sent
  // rows' ids go to d_sent_orig + k * max_batch -- fixed regions, so the host needs no plan.
  dycl_status rebalance_device(Tensor t, int* cnt_slot, const Shape& sh, int orig_cur) {
    const int k = (int)drb.size();
    if (k >= dycl::DRB_MAX_LEVELS) return fail(g, DYCL_E_UNSUPPORTED, "device rebalancing: too many levels");
    if (!g->drb_win) {
      std::string err;
      if (!g->tr->window(g->drb_bytes, &g->drb_win, &g->drb_peers, &err)) return fail(g, DYCL_E_NCCL, err);
    }
    dycl::DrbArgs a{};
    a.rank = g->tr->rank;
    a.world = g->tr->world;
    a.level = k;
    a.max_rows = (int)g->max_batch;
    a.K = g->K;
    a.peers = g->drb_peers;
    a.rows_off = g->drb_rows_off;
    a.ret_off = g->drb_ret_off;
    a.epoch = g->d_drb_epoch;
    a.err = g->d_drb_err;
    a.ticket = g->d_drb_ticket;
    a.plan = g->d_drb_plan;
    a.cnt = cnt_slot;
    a.plane_b = t.b >= 0 ? reinterpret_cast<uint8_t*>(g->buf[t.b]) : nullptr;
    a.plane_f = t.f >= 0 ? reinterpret_cast<uint8_t*>(g->buf32[t.f]) : nullptr;
    a.plane_b_bytes = t.b >= 0 ? sh.row_elems() * 2 : 0;
    a.plane_f_bytes = t.f >= 0 ? sh.row_elems() * (g->stream_pair ? 2 : 4) : 0;
    a.row_bytes = a.plane_b_bytes + a.plane_f_bytes;
    if (a.row_bytes + 16 > (long long)((g->drb_ret_off - g->drb_rows_off) / g->max_batch))
      return fail(g, DYCL_E_STATE, "device rebalancing: row larger than the window's row slots");
    a.orig = g->d_orig[orig_cur];
    a.sent_orig = g->d_sent_orig + (size_t)k * g->max_batch;
    a.gid_base = global_offset;
    a.own = own;
    a.ext0 = (int)(g->max_batch * (1 + k));
    a.ext_gid = g->d_ext_gid;
    a.res_path = out_path;
    a.res_margin = out_margin;
    a.res_logits = out_logits;
    cudaError_t e = dycl::drb_counts(a, st);
    if (e == cudaSuccess) e = dycl::drb_push(a, g->num_sms, st);
    if (e == cudaSuccess) e = dycl::drb_wait(a, 0, st);
    if (e == cudaSuccess) e = dycl::drb_pull(a, g->num_sms, st);
    if (e != cudaSuccess) return cuda_fail(g, e, "device rebalancing");
    nlaunch += 4;
    drb.push_back(a);
    batch = (int)g->max_batch;                     // rows held are known on the device only
    return DYCL_OK;
  }

  dycl_status return_results_device() {
    for (int k = (int)drb.size() - 1; k >= 0; --k) {
      const dycl::DrbArgs& a = drb[k];
      cudaError_t e = dycl::drb_ret_push(a, g->num_sms, st);
      if (e == cudaSuccess) e = dycl::drb_wait(a, 1, st);
      if (e == cudaSuccess) e = dycl::drb_ret_pull(a, g->num_sms, st);
      if (e != cudaSuccess) return cuda_fail(g, e, "device rebalancing (return)");
      nlaunch += 3;
    }
    g->drb_levels_last = (int)drb.size();
    return DYCL_OK;
  }

  dycl_status rebalance(Tensor t, int* cnt_slot, const Shape& sh, int orig_cur) {
    if (g->rb_device) return rebalance_device(t, cnt_slot, sh, orig_cur);
    dycl::Transport* T = g->tr;
    const int W = T->world, me = T->rank;
    std::vector<int> counts(W);
    std::string err;
    if (!T->allgather_int(cnt_slot, counts.data(), st, &err)) return fail(g, DYCL_E_NCCL, err);
    Level L;
    L.send.assign(W, 0);
    L.recv.assign(W, 0);
    int newc = 0;
    if (dycl_rebalance_plan(counts.data(), W, me, L.send.data(), L.recv.data(), &newc) != DYCL_OK)
      return fail(g, DYCL_E_INVALID_ARG, "rebalance plan");
    long long moved = 0;
    for (int r = 0; r < W; ++r) {
      std::vector<int> sd(W), rc(W);
      int nc = 0;
      dycl_rebalance_plan(counts.data(), W, r, sd.data(), rc.data(), &nc);
      for (int j = 0; j < W; ++j) moved += sd[j];
    }
    for (int j = 0; j < W; ++j) {
      L.n_send += L.send[j];
      L.n_recv += L.recv[j];
    }
    if (newc > g->max_batch) return fail(g, DYCL_E_SHAPE_MISMATCH, "rebalance: rows held exceed max_batch");
    L.ext0 = own + ext_used;
    L.sent0 = sent_used;
    L.moved_any = moved > 0;
    if (moved == 0) {                                // nobody moves: no exchange, no return
      levels.push_back(L);
      return DYCL_OK;
    }
    if (ext_used + L.n_recv > g->rb_rows - own || sent_used + L.n_send > g->rb_rows)
      return fail(g, DYCL_E_STATE, "rebalance: result space exhausted");
    const int s_own = counts[me], keep = s_own - L.n_send;
    int32_t* meta_send = g->d_meta;
    int32_t* meta_recv = g->d_meta + 4 * (size_t)g->max_batch;
    int* orig = g->d_orig[orig_cur];
    cudaError_t e = dycl::launch_rb_pack(orig, keep, L.n_send, out_path, out_margin, g->d_ext_gid, global_offset, own,
                                         g->d_sent_orig + sent_used, meta_send, st);
    if (e != cudaSuccess) return cuda_fail(g, e, "launch_rb_pack");
    std::vector<dycl::Transport::Msg> sends, recvs;
    const size_t rb = (size_t)sh.row_elems() * 2, rf = (size_t)sh.row_elems() * (g->stream_pair ? 2 : 4);
    int so = keep, ro = s_own;                       // row cursors (destination / source rank ascending)
    for (int j = 0; j < W; ++j) {
      if (L.send[j]) {
        if (t.b >= 0) sends.push_back({j, (char*)g->buf[t.b] + so * rb, L.send[j] * rb});
        if (t.f >= 0) sends.push_back({j, (char*)g->buf32[t.f] + so * rf, L.send[j] * rf});
        sends.push_back({j, meta_send + 4 * (size_t)(so - keep), (size_t)L.send[j] * 16});
        so += L.send[j];
      }
      if (L.recv[j]) {
        if (t.b >= 0) recvs.push_back({j, (char*)g->buf[t.b] + ro * rb, L.recv[j] * rb});
        if (t.f >= 0) recvs.push_back({j, (char*)g->buf32[t.f] + ro * rf, L.recv[j] * rf});
        recvs.push_back({j, meta_recv + 4 * (size_t)(ro - s_own), (size_t)L.recv[j] * 16});
        ro += L.recv[j];
      }
    }
    if (!T->exchange(sends, recvs, st, &err)) return fail(g, DYCL_E_NCCL, err);
    e = dycl::launch_rb_unpack(orig, s_own, L.n_recv, L.ext0, own, meta_recv, out_path, out_margin, g->d_ext_gid, st);
    if (e == cudaSuccess) e = dycl::launch_set_int(cnt_slot, newc, st);
    if (e != cudaSuccess) return cuda_fail(g, e, "rebalance unpack");
    ext_used += L.n_recv;
    sent_used += L.n_send;
    g->rb_sent += L.n_send;
    g->rb_recv += L.n_recv;
    if (newc > batch) batch = newc;                  // grid sizing for the rows now held
    levels.push_back(L);
    return DYCL_OK;
  }

  // End of run: results of rows computed away from home go back by the reverse plans, last
  // level first (a row forwarded twice returns through its intermediate rank), and are
  // scattered to their result-space id; own rows then reach the caller's buffers.
  dycl_status return_results() {
    if (g->tr && g->rb_device) return return_results_device();
    if (!g->tr || levels.empty()) return DYCL_OK;
    const int K = g->K, W = g->tr->world;
    std::string err;
    for (int li = (int)levels.size() - 1; li >= 0; --li) {
      const Level& L = levels[li];
      if (!L.moved_any) continue;                    // every rank knows every plan: all skip together
      std::vector<dycl::Transport::Msg> sends, recvs;
      int ro = L.ext0;
      long long so = L.sent0;
      for (int j = 0; j < W; ++j) {
        if (L.recv[j]) {                             // results of rows received from j go back to j
          sends.push_back({j, out_logits + (size_t)ro * K, (size_t)L.recv[j] * K * 4});
          sends.push_back({j, out_path + ro, (size_t)L.recv[j] * 4});
          sends.push_back({j, out_margin + ro, (size_t)L.recv[j] * 4});
          ro += L.recv[j];
        }
        if (L.send[j]) {
          const long long k = so - L.sent0;
          recvs.push_back({j, g->d_ret_logits + (size_t)k * K, (size_t)L.send[j] * K * 4});
          recvs.push_back({j, g->d_ret_path + k, (size_t)L.send[j] * 4});
          recvs.push_back({j, g->d_ret_margin + k, (size_t)L.send[j] * 4});
          so += L.send[j];
        }
      }
      if (!g->tr->exchange(sends, recvs, st, &err)) return fail(g, DYCL_E_NCCL, err);
      cudaError_t e = dycl::launch_rb_return(g->d_sent_orig + L.sent0, L.n_send, K, g->d_ret_logits, g->d_ret_path,
                                             g->d_ret_margin, out_logits, out_path, out_margin, st);
      if (e != cudaSuccess) return cuda_fail(g, e, "launch_rb_return");
    }
    return DYCL_OK;
  }
};

}  // namespace

// =================================================================== C ABI
extern "C" {

dycl_status dycl_graph_create(int cuda_device, int in_h, int in_w, int in_c, dycl_graph* out) {
  if (!out || in_h <= 0 || in_w <= 0 || in_c <= 0) return fail(nullptr, DYCL_E_INVALID_ARG, "bad argument");
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(nullptr, DYCL_E_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  if (cuda_device < 0 || cuda_device >= ndev) return fail(nullptr, DYCL_E_INVALID_ARG, "bad device index");
  dycl_graph g = new (std::nothrow) dycl_graph_s();
  if (!g) return fail(nullptr, DYCL_E_OOM, "host allocation failed");
  g->device = cuda_device;
  g->input = Shape{in_h, in_w, in_c};
  if (const char* cp = getenv("DYCL_CONV_PATH")) g->conv_path = atoi(cp);
  if (const char* cd = getenv("DYCL_CONV_DBG")) g->conv_dbg = atoi(cd);
  if (const char* hk = getenv("DYCL_HALO_KSKIP")) g->halo_kskip = atoi(hk);
  if (const char* nf = getenv("DYCL_NO_FUSE")) g->no_fuse = atoi(nf);
  if (const char* hc = getenv("DYCL_HEAD_CUDA_CORE")) g->head_cuda_core = atoi(hc);
  if (const char* mf = getenv("DYCL_MAX_FUSE")) g->max_fuse = atoi(mf);
  if (const char* ni = getenv("DYCL_NO_INPLACE")) g->no_inplace = atoi(ni);
  if (const char* nz = getenv("DYCL_NO_ZERO_COPY")) g->no_zero_copy = atoi(nz);
  if (const char* zm = getenv("DYCL_ZC_PROJ_MIN")) g->zc_proj_min = std::max(dycl::ZC_MIN_ROWS, atoi(zm));
  if (const char* ug = getenv("DYCL_GRAPH")) g->use_graph = atoi(ug) != 0;
  if (getenv("DYCL_TS")) {
    cudaMalloc(&g->dbg_ts, 8 * 16 * sizeof(long long));
    g->dbg_ts_pick = atoi(getenv("DYCL_TS")) > 1 ? atoi(getenv("DYCL_TS")) : 0;
    if (getenv("DYCL_TS_CONV")) {
      g->dbg_ts_conv = atoi(getenv("DYCL_TS_CONV"));
      g->dbg_ts_pick = -1;                         // no fused-block launch records
    }
    cudaMemset(g->dbg_ts, 0, 8 * 16 * sizeof(long long));
  }
  cudaSetDevice(cuda_device);
  cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, cuda_device);
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, cuda_device);
  if (major != 10) {
    delete g;
    return fail(nullptr, DYCL_E_UNSUPPORTED, "libdycl is built for sm_100a (B200) only");
  }
  *out = g;
  return DYCL_OK;
}

dycl_status dycl_graph_destroy(dycl_graph g) {
  if (!g) return DYCL_OK;
  cudaSetDevice(g->device);
  for (Subnet& s : g->subnets)
    for (Layer& L : s.layers) {
      cudaFree(L.d_w);
      cudaFree(L.d_wrt);
      cudaFree(L.d_wt);
      cudaFree(L.d_w2);
      cudaFree(L.d_b2);
      cudaFree(L.d_wcat);
      cudaFree(L.d_bcat);
      cudaFree(L.d_b);
    }
  for (auto* b : g->buf) cudaFree(b);
  for (auto* b : g->buf32) cudaFree(b);
  cudaFree(g->d_counts);
  cudaFree(g->d_orig[0]);
  cudaFree(g->d_orig[1]);
  cudaFree(g->d_list1);
  cudaFree(g->d_list0);
  cudaFree(g->d_flag);
  cudaFree(g->d_pred);
  cudaFree(g->d_z);
  cudaFree(g->d_gpool);
  cudaFree(g->d_a2);
  cudaFree(g->d_rnn_w);
  cudaFree(g->d_rnn_state);
  for (Node& N : g->nodes) cudaFree(N.d_w_out);
  cudaFree(g->d_gap_part);
  cudaFree(g->d_gap_pooled);
  for (auto* p : g->d_pool32) cudaFree(p);
  cudaFree(g->d_in_stage);
  cudaFree(g->d_logit_stage);
  cudaFree(g->d_path_stage);
  cudaFree(g->d_margin_stage);
  cudaFree(g->dbg_ts);
  cudaFree(g->d_drb_plan);
  cudaFree(g->d_drb_epoch);
  cudaFree(g->d_drb_err);
  cudaFree(g->d_drb_ticket);
  cudaFree(g->d_res_logits);
  cudaFree(g->d_res_path);
  cudaFree(g->d_res_margin);
  cudaFree(g->d_ext_gid);
  cudaFree(g->d_sent_orig);
  cudaFree(g->d_meta);
  cudaFree(g->d_ret_logits);
  cudaFree(g->d_ret_path);
  cudaFree(g->d_ret_margin);
  delete g->tr;
  for (auto& e : g->graphs)
    if (e.exec) cudaGraphExecDestroy(e.exec);
  if (g->cap_stream) cudaStreamDestroy(g->cap_stream);
  if (g->h2d_stream) cudaStreamDestroy(g->h2d_stream);
  if (g->d2h_stream) cudaStreamDestroy(g->d2h_stream);
  for (int i = 0; i < 2; ++i) {
    if (g->ev_h2d[i]) cudaEventDestroy(g->ev_h2d[i]);
    if (g->ev_run[i]) cudaEventDestroy(g->ev_run[i]);
    if (g->ev_d2h[i]) cudaEventDestroy(g->ev_d2h[i]);
  }
  for (auto& L : g->prof) {
    cudaEventDestroy(L.e0);
    cudaEventDestroy(L.e1);
  }
  delete g;
  return DYCL_OK;
}

const char* dycl_last_error(dycl_graph g) { return g ? g->err.c_str() : g_create_err.c_str(); }

dycl_status dycl_graph_set_precision(dycl_graph g, int precision) {
  if (!g) return DYCL_E_INVALID_ARG;
  if (g->finalized) return fail(g, DYCL_E_STATE, "graph already finalized");
  if (precision == DYCL_PREC_BF16X3_PARITY)
    return fail(g, DYCL_E_UNSUPPORTED, "BF16X3 parity mode is implemented for the generative graph (dycl_s2s); "
                                       "image graphs meet decision parity in FP32_STREAM (DESIGN.md R13)");
  if (precision != DYCL_PREC_BF16 && precision != DYCL_PREC_FP32_STREAM)
    return fail(g, DYCL_E_INVALID_ARG, "unknown precision mode");
  g->precision = precision;
  return DYCL_OK;
}

dycl_status dycl_subnet_begin(dycl_graph g, dycl_node* out) {
  if (!g || !out) return DYCL_E_INVALID_ARG;
  if (g->finalized) return fail(g, DYCL_E_STATE, "graph already finalized");
  g->subnets.emplace_back();
  *out = (dycl_node)g->subnets.size() - 1;
  return DYCL_OK;
}

dycl_status dycl_subnet_block_begin(dycl_graph g, dycl_node sn) {
  if (dycl_status s = check_sn(g, sn)) return s;
  Layer L;
  L.kind = L_BLOCK;
  g->subnets[sn].layers.push_back(std::move(L));
  return DYCL_OK;
}

dycl_status dycl_subnet_conv2d(dycl_graph g, dycl_node sn, int c_in, int c_out, int k, int stride, int pad,
                               const uint16_t* w_bf16, const float* bias, dycl_act act, int residual) {
  if (dycl_status s = check_sn(g, sn)) return s;
  if (!w_bf16 || !bias || c_in <= 0 || c_out <= 0 || k < 1 || k > 7 || (stride != 1 && stride != 2) || pad < 0 ||
      pad >= k || (act != DYCL_ACT_NONE && act != DYCL_ACT_RELU))
    return fail(g, DYCL_E_INVALID_ARG, "conv2d: bad argument");
  if (c_out % 16) return fail(g, DYCL_E_UNSUPPORTED, "conv2d: c_out must be a multiple of 16");
  Layer L;
  L.kind = L_CONV;
  L.cout = c_out; L.k = k; L.stride = stride; L.pad = pad;
  L.relu = act == DYCL_ACT_RELU;
  L.residual = residual ? 1 : 0;
  L.w.assign(w_bf16, w_bf16 + (size_t)c_out * k * k * c_in);
  L.b.assign(bias, bias + c_out);
  g->subnets[sn].layers.push_back(std::move(L));
  return DYCL_OK;
}

dycl_status dycl_subnet_dense(dycl_graph g, dycl_node sn, int n_in, int n_out, const uint16_t* w_bf16,
                              const float* bias, dycl_act act, int out_fp32) {
  if (dycl_status s = check_sn(g, sn)) return s;
  if (!w_bf16 || !bias || n_in <= 0 || n_out <= 0 || (act != DYCL_ACT_NONE && act != DYCL_ACT_RELU))
    return fail(g, DYCL_E_INVALID_ARG, "dense: bad argument");
  if (!out_fp32 && n_out % 16) return fail(g, DYCL_E_UNSUPPORTED, "dense: bf16 n_out must be a multiple of 16");
  if (out_fp32 && act != DYCL_ACT_NONE) return fail(g, DYCL_E_UNSUPPORTED, "dense: fp32 heads take no activation");
  Layer L;
  L.kind = L_DENSE;
  L.cout = n_out;
  L.relu = act == DYCL_ACT_RELU;
  L.out_fp32 = out_fp32 ? 1 : 0;
  L.w.assign(w_bf16, w_bf16 + (size_t)n_out * n_in);
  L.b.assign(bias, bias + n_out);
  g->subnets[sn].layers.push_back(std::move(L));
  return DYCL_OK;
}

dycl_status dycl_subnet_projection(dycl_graph g, dycl_node sn, int c_in, int c_out, int stride,
                                   const uint16_t* w_bf16, const float* bias) {
  if (dycl_status s = check_sn(g, sn)) return s;
  if (!w_bf16 || !bias || c_in <= 0 || c_out <= 0 || stride < 1 || stride > 2)
    return fail(g, DYCL_E_INVALID_ARG, "projection: bad argument");
  if (c_out % 16) return fail(g, DYCL_E_UNSUPPORTED, "projection: c_out must be a multiple of 16");
  Layer L;
  L.kind = L_PROJ;
  L.cout = c_out; L.k = 1; L.stride = stride; L.pad = 0;
  L.w.assign(w_bf16, w_bf16 + (size_t)c_out * c_in);
  L.b.assign(bias, bias + c_out);
  g->subnets[sn].layers.push_back(std::move(L));
  return DYCL_OK;
}

dycl_status dycl_subnet_maxpool(dycl_graph g, dycl_node sn, int k, int stride, int pad) {
  if (dycl_status s = check_sn(g, sn)) return s;
  if (k < 1 || k > 7 || stride < 1 || stride > 4 || pad < 0 || pad >= k)
    return fail(g, DYCL_E_INVALID_ARG, "maxpool: bad argument");
  Layer L;
  L.kind = L_MAXPOOL;
  L.k = k; L.stride = stride; L.pad = pad;
  g->subnets[sn].layers.push_back(std::move(L));
  return DYCL_OK;
}

dycl_status dycl_subnet_gap(dycl_graph g, dycl_node sn) {
  if (dycl_status s = check_sn(g, sn)) return s;
  Layer L;
  L.kind = L_GAP;
  g->subnets[sn].layers.push_back(std::move(L));
  return DYCL_OK;
}

dycl_status dycl_subnet_end(dycl_graph g, dycl_node sn) {
  if (dycl_status s = check_sn(g, sn)) return s;
  if (g->subnets[sn].layers.empty()) return fail(g, DYCL_E_INVALID_ARG, "empty subnet");
  g->subnets[sn].ended = true;
  return DYCL_OK;
}

static dycl_status add_node(dycl_graph g, Node N, bool needs_head_sn) {
  if (!g) return DYCL_E_INVALID_ARG;
  if (g->finalized) return fail(g, DYCL_E_STATE, "graph already finalized");
  const int ns = (int)g->subnets.size();
  if (N.sn < 0 || N.sn >= ns || (N.kind == N_GATE && (N.then_sn < 0 || N.then_sn >= ns)))
    return fail(g, DYCL_E_INVALID_ARG, "bad subnet id");
  if (!g->subnets[N.sn].ended || (N.kind == N_GATE && !g->subnets[N.then_sn].ended))
    return fail(g, DYCL_E_STATE, "subnet not ended");
  if (!g->nodes.empty() && g->nodes.back().kind == N_FINAL)
    return fail(g, DYCL_E_STATE, "no node may follow dycl_final");
  (void)needs_head_sn;
  g->nodes.push_back(N);
  return DYCL_OK;
}

dycl_status dycl_seq(dycl_graph g, dycl_node subnet) {
  Node N{};
  N.kind = N_SEQ;
  N.sn = subnet;
  return add_node(g, N, false);
}

dycl_status dycl_exit(dycl_graph g, dycl_node head_subnet, float tau) {
  Node N{};
  N.kind = N_EXIT;
  N.sn = head_subnet;
  N.thr = tau;
  dycl_status s = add_node(g, N, true);
  if (s == DYCL_OK) g->nodes.back().ordinal = g->n_exits++;
  return s;
}

dycl_status dycl_gate(dycl_graph g, dycl_node gate_subnet, float thr, dycl_node then_subnet) {
  Node N{};
  N.kind = N_GATE;
  N.sn = gate_subnet;
  N.then_sn = then_subnet;
  N.thr = thr;
  if (g && g->n_gates >= 31) return fail(g, DYCL_E_UNSUPPORTED, "at most 31 gates (path word bits)");
  dycl_status s = add_node(g, N, true);
  if (s == DYCL_OK) g->nodes.back().ordinal = g->n_gates++;
  return s;
}

dycl_status dycl_rnn_cell(dycl_graph g, int n_in, int hidden, const float* w_ih, const float* w_hh,
                          const float* b_ih, const float* b_hh) {
  if (!g) return DYCL_E_INVALID_ARG;
  if (g->finalized) return fail(g, DYCL_E_STATE, "graph already finalized");
  if (g->rnn_hidden) return fail(g, DYCL_E_STATE, "the graph already has an RNN cell");
  if (n_in < 1 || n_in > 16 || hidden < 1 || hidden > 16 || !w_ih || !w_hh || !b_ih || !b_hh)
    return fail(g, DYCL_E_INVALID_ARG, "rnn cell: 1 <= n_in, hidden <= 16, non-null weights");
  const size_t H4 = 4 * (size_t)hidden;
  g->rnn_w.assign(w_ih, w_ih + H4 * n_in);
  g->rnn_w.insert(g->rnn_w.end(), w_hh, w_hh + H4 * hidden);
  g->rnn_w.insert(g->rnn_w.end(), b_ih, b_ih + H4);
  g->rnn_w.insert(g->rnn_w.end(), b_hh, b_hh + H4);
  g->rnn_in = n_in;
  g->rnn_hidden = hidden;
  return DYCL_OK;
}

dycl_status dycl_gate_rnn(dycl_graph g, dycl_node proj_subnet, const float* w_out, float b_out, float thr,
                          dycl_node then_subnet) {
  if (!g) return DYCL_E_INVALID_ARG;
  if (!g->rnn_hidden) return fail(g, DYCL_E_STATE, "dycl_gate_rnn before dycl_rnn_cell");
  if (!w_out) return fail(g, DYCL_E_INVALID_ARG, "null w_out");
  Node N{};
  N.kind = N_GATE;
  N.sn = proj_subnet;
  N.then_sn = then_subnet;
  N.thr = thr;
  N.rnn = 1;
  N.w_out.assign(w_out, w_out + g->rnn_hidden);
  N.b_out = b_out;
  if (g->n_gates >= 31) return fail(g, DYCL_E_UNSUPPORTED, "at most 31 gates (path word bits)");
  dycl_status s = add_node(g, N, true);
  if (s == DYCL_OK) g->nodes.back().ordinal = g->n_gates++;
  return s;
}

dycl_status dycl_final(dycl_graph g, dycl_node head_subnet) {
  Node N{};
  N.kind = N_FINAL;
  N.sn = head_subnet;
  return add_node(g, N, true);
}

dycl_status dycl_finalize(dycl_graph g, int64_t max_batch) {
  if (!g) return DYCL_E_INVALID_ARG;
  if (g->finalized) return fail(g, DYCL_E_STATE, "graph already finalized");
  if (max_batch <= 0 || max_batch > (1 << 26)) return fail(g, DYCL_E_INVALID_ARG, "bad max_batch");
  if (g->nodes.empty() || g->nodes.back().kind != N_FINAL)
    return fail(g, DYCL_E_STATE, "the chain must end with dycl_final");
  CK(cudaSetDevice(g->device));
  // ---- Alg. 2: propagate the per-sample shape along the chain from N0
  Shape cur = g->input;
  long long maxrow = cur.row_elems();
  std::vector<int> planned(g->subnets.size(), 0);
  std::vector<Shape> planned_in(g->subnets.size());
  auto plan = [&](int sn, const Shape& in) -> dycl_status {
    if (planned[sn]) {
      if (!(planned_in[sn] == in)) return fail(g, DYCL_E_SHAPE_MISMATCH, "subnet reused with a different input shape");
      return DYCL_OK;
    }
    dycl_status s = plan_subnet(g, g->subnets[sn], in, sn);
    if (s) return s;
    // registration-time c_in / n_in must agree with propagated shapes
    for (const Layer& L : g->subnets[sn].layers) {
      if ((L.kind == L_CONV || L.kind == L_PROJ) && (long long)L.w.size() != (long long)L.cout * L.k * L.k * L.in.C)
        return fail(g, DYCL_E_SHAPE_MISMATCH, "conv2d c_in disagrees with the propagated shape");
      if (L.kind == L_DENSE && (long long)L.w.size() != (long long)L.cout * L.in.C)
        return fail(g, DYCL_E_SHAPE_MISMATCH, "dense n_in disagrees with the propagated shape");
      maxrow = std::max(maxrow, L.out.row_elems());
    }
    planned[sn] = 1;
    planned_in[sn] = in;
    return DYCL_OK;
  };
  g->K = 0;
  for (Node& N : g->nodes) {
    N.in = cur;
    dycl_status s = plan(N.sn, cur);
    if (s) return s;
    const Subnet& S = g->subnets[N.sn];
    if (N.kind == N_SEQ) {
      if (S.is_head) return fail(g, DYCL_E_UNSUPPORTED, "dycl_seq on a head subnet");
      cur = S.out;
    } else {
      if (!S.is_head) return fail(g, DYCL_E_SHAPE_MISMATCH, "exit/gate/final need a [gap] + dense(out_fp32) head");
      if (S.in.Cp() % 8 || S.in.Cp() / 8 > 256) return fail(g, DYCL_E_UNSUPPORTED, "head input channels");
      if (N.kind == N_GATE) {
        if (N.rnn ? S.head_K != g->rnn_in : S.head_K != 1)
          return fail(g, N.rnn ? DYCL_E_SHAPE_MISMATCH : DYCL_E_SIGNATURE,
                      N.rnn ? "rnn gate: proj output width != the cell's n_in" : "gate head must produce one logit");
        if ((s = plan(N.then_sn, cur))) return s;
        const Subnet& T = g->subnets[N.then_sn];
        if (T.is_head) return fail(g, DYCL_E_UNSUPPORTED, "gate then-branch is a head");
        if (T.out == cur) N.skip_mode = 0;
        else if (T.out.H * 2 == cur.H && T.out.W * 2 == cur.W && T.out.C == 2 * cur.C && cur.C % 16 == 0)
          N.skip_mode = 1;
        else return fail(g, DYCL_E_SHAPE_JOIN, "gate: then-branch output shape joins neither identity nor option A");
        cur = T.out;
      } else {
        if (g->K == 0) g->K = S.head_K;
        else if (g->K != S.head_K) return fail(g, DYCL_E_SIGNATURE, "exit/final heads disagree on K");
      }
    }
    N.out = cur;
    maxrow = std::max(maxrow, cur.row_elems());
  }
  // ---- activation layout: NHWC when every conv past an (at most 8-channel) input has 64-multiple
  // channel counts (the im2col GEMM's operand boxes are 64 channels wide) and no gate needs an
  // option-A skip copy; channel-planar otherwise (the CIFAR-width kernels).
  {
    bool ok = g->input.Cp() == 8;
    // per-tensor rule (Exec::lay): C % 64 == 0 tensors are NHWC; a conv reading one runs on the
    // im2col GEMM, so its output width must be a multiple of 64 too (else: planar graph)
    for (size_t i = 0; i < g->subnets.size() && ok; ++i)
      if (planned[i])
        for (const Layer& L : g->subnets[i].layers)
          if ((L.kind == L_CONV || L.kind == L_PROJ) && L.in.Cp() % 64 == 0 && !(L.in.H == 1 && L.in.W == 1)) {
            ok = ok && L.out.C % 64 == 0 && (L.res_mode != 2 || (L.res_shape.Cp() % 4 == 0));
          }
    const char* env = getenv("DYCL_NHWC");
    g->nhwc = ok && !(env && atoi(env) == 0);
    // pair residual stream (see stream_pair): NHWC, fp32-stream precision, no gates (in-place gate
    // forms read the fp32 copy), no dense trunk layers or SMEM-fused basic blocks, and no max pool
    // whose fp32 output copy a block would read as its identity shortcut
    bool pair = g->nhwc && g->precision == DYCL_PREC_FP32_STREAM && g->n_gates == 0 && !getenv("DYCL_NO_PAIR");
    for (size_t i = 0; i < g->subnets.size() && pair; ++i) {
      if (!planned[i]) continue;
      const auto& Ls = g->subnets[i].layers;
      for (size_t li = 0; li < Ls.size() && pair; ++li) {
        const Layer& L = Ls[li];
        if (L.kind == L_DENSE && !L.out_fp32) pair = false;
        if (L.kind == L_BLOCK && li + 2 < Ls.size() && Ls[li + 1].kind == L_CONV && Ls[li + 1].k == 3 &&
            Ls[li + 2].kind == L_CONV && Ls[li + 2].k == 3 &&
            dycl::block_fused_eligible(Ls[li + 1].in.C, Ls[li + 1].in.H, Ls[li + 1].in.W))
          pair = false;
        if (L.kind == L_MAXPOOL) {
          bool proj = false;
          if (li + 1 < Ls.size() && Ls[li + 1].kind == L_BLOCK)
            for (size_t lj = li + 2; lj < Ls.size() && Ls[lj].kind != L_BLOCK; ++lj) proj = proj || Ls[lj].kind == L_PROJ;
          if (li + 1 == Ls.size() || (Ls[li + 1].kind == L_BLOCK && !proj)) pair = false;
        }
      }
    }
    g->stream_pair = pair;
    // space-to-depth stem: the first layer run is a 7x7 / stride-2 / pad-3 conv on <= 4 input
    // channels followed by a 3x3 / stride-2 / pad-1 max pool (the ImageNet ResNet stem)
    g->stem_s4d = 0;
    const char* env4 = getenv("DYCL_STEM_S4D");
    if (g->nhwc && !(env4 && atoi(env4) == 0)) {
      Subnet& S0 = g->subnets[g->nodes[0].sn];
      if (S0.layers.size() >= 2) {
        Layer &L0 = S0.layers[0], &L1 = S0.layers[1];
        if (L0.kind == L_CONV && L0.k == 7 && L0.stride == 2 && L0.pad == 3 && L0.in.C <= 4 && !L0.residual &&
            L0.relu && L0.in.H % 4 == 0 && L0.in.W % 4 == 0 && L0.out.H * 2 == L0.in.H && L0.out.W * 2 == L0.in.W &&
            L1.kind == L_MAXPOOL && L1.k == 3 && L1.stride == 2 && L1.pad == 1 && L0.cout % 16 == 0) {
          // the 2x2 form on the halo kernel measured slower end to end (stem 2.37 vs 2.2 ms, and the
          // plain NHWC max pool 1.9 vs 0.9 ms per 2048-row chunk): opt-in DYCL_STEM_S2D2=1
          const char* env2 = getenv("DYCL_STEM_S2D2");
          if (env2 && atoi(env2) == 1 && L0.cout == 64 && L0.in.C <= 4) {
            L0.s2d2 = 1;                    // the halo-tile form; the max pool reads plain NHWC
            g->stem_s2d2 = 1;
          } else {
            L0.s4d = 1;
            L1.pool_s2d = 1;
            g->stem_s4d = 1;
          }
        }
      }
    }
  }
  // ---- which subnets read their input's fp32 stream copy: a leading block with an identity
  // shortcut (conv residual, no projection) or a max pool; conservative otherwise
  for (Subnet& S : g->subnets) {
    S.needs_in32 = true;
    if (S.layers.empty() || S.is_head) continue;
    const Layer& L0 = S.layers[0];
    if (L0.kind == L_CONV || L0.kind == L_DENSE) {
      S.needs_in32 = false;                      // a plain first layer reads the bf16 operand copy
    } else if (L0.kind == L_BLOCK) {
      bool proj = false, res = false;
      for (size_t li = 1; li < S.layers.size() && S.layers[li].kind != L_BLOCK; ++li) {
        proj = proj || S.layers[li].kind == L_PROJ;
        res = res || S.layers[li].residual;
        if (S.layers[li].kind != L_CONV && S.layers[li].kind != L_PROJ) res = true;   // anything else: keep
      }
      S.needs_in32 = res && !proj;
    }
  }
  // ---- weights -> HBM (snapshot), workspace for max_batch
  for (size_t i = 0; i < g->subnets.size(); ++i)
    if (planned[i])
      if (dycl_status s = upload_subnet(g, g->subnets[i])) return s;
  g->max_batch = max_batch;
  g->max_row_elems = maxrow;
  const size_t nb = (size_t)max_batch;
  for (auto& b : g->buf)
    if (dycl_status s = dmalloc(g, &b, nb * (size_t)maxrow * 2)) return s;
  if (g->precision == DYCL_PREC_FP32_STREAM)
    for (auto& b : g->buf32)
      if (dycl_status s = dmalloc(g, &b, nb * (size_t)maxrow * 4)) return s;
  g->n_slots = 1 + 2 * (int)g->nodes.size();
  if (dycl_status s = dmalloc(g, &g->d_counts, g->n_slots * sizeof(int))) return s;
  CK(cudaMemset(g->d_counts, 0, g->n_slots * sizeof(int)));
  for (auto& o : g->d_orig)
    if (dycl_status s = dmalloc(g, &o, nb * 4)) return s;
  if (dycl_status s = dmalloc(g, &g->d_list1, nb * 4)) return s;
  if (dycl_status s = dmalloc(g, &g->d_list0, nb * 4)) return s;
  if (dycl_status s = dmalloc(g, &g->d_flag, nb)) return s;
  if (dycl_status s = dmalloc(g, &g->d_pred, nb * 4)) return s;
  if (g->rnn_hidden && g->K < g->rnn_in) return fail(g, DYCL_E_UNSUPPORTED, "rnn cell n_in exceeds the head width K");
  if (dycl_status s = dmalloc(g, &g->d_z, nb * (size_t)std::max(g->K, 1) * 4)) return s;
  if (g->rnn_hidden) {
    if (dycl_status s = dmalloc(g, &g->d_rnn_w, g->rnn_w.size() * 4)) return s;
    CK(cudaMemcpy(g->d_rnn_w, g->rnn_w.data(), g->rnn_w.size() * 4, cudaMemcpyHostToDevice));
    if (dycl_status s = dmalloc(g, &g->d_rnn_state, nb * 2 * g->rnn_hidden * 4)) return s;
    for (Node& N : g->nodes)
      if (N.rnn) {
        if (dycl_status s = dmalloc(g, &N.d_w_out, N.w_out.size() * 4)) return s;
        CK(cudaMemcpy(N.d_w_out, N.w_out.data(), N.w_out.size() * 4, cudaMemcpyHostToDevice));
      }
  }
  if (g->precision == DYCL_PREC_FP32_STREAM) {
    bool fused_any = false;
    for (size_t i = 0; i < g->subnets.size(); ++i)
      if (planned[i])
        for (const Layer& L : g->subnets[i].layers)
          fused_any = fused_any || (L.kind == L_CONV && L.d_wrt && dycl::block_fused_eligible(L.in.C, L.in.H, L.in.W));
    if (fused_any)
      for (auto& p : g->d_pool32)
        if (dycl_status s = dmalloc(g, &p, nb * 32 * 4)) return s;
  }
  {
    int cmax = 0;
    for (const Node& N : g->nodes)
      if (N.kind != N_SEQ && g->subnets[N.sn].layers.back().d_wt) cmax = std::max(cmax, g->subnets[N.sn].in.Cp());
    if (cmax > 0)
      if (dycl_status s = dmalloc(g, &g->d_gpool, nb * (size_t)cmax * 4)) return s;
    if (cmax > 0 && !g->head_cuda_core)
      if (dycl_status s = dmalloc(g, &g->d_a2, nb * (size_t)cmax * 2 * 2)) return s;
  }
  {
    // conv_gemm fused GAP: the last conv of a sub-network that feeds an exit / final head
    size_t part = 0, pooled = 0;
    for (size_t ni = 0; ni + 1 < g->nodes.size(); ++ni) {
      const Node& N = g->nodes[ni];
      if (N.kind != N_SEQ || (g->nodes[ni + 1].kind != N_EXIT && g->nodes[ni + 1].kind != N_FINAL)) continue;
      const Subnet& S = g->subnets[N.sn];
      if (S.layers.empty() || S.layers.back().kind != L_CONV) continue;
      const Layer& L = S.layers.back();
      const int hw = L.out.H * L.out.W;
      if (!g->nhwc || L.out.C % 64 || L.in.Cp() % 64 || hw < 32 || 4.0 * L.out.row_elems() < 128 * 1024 ||
          gap_group(hw) < 4)
        continue;
      part = std::max(part, (size_t)nb * (hw / gap_group(hw)) * L.out.C);
      pooled = std::max(pooled, (size_t)nb * L.out.C);
    }
    if (part && !getenv("DYCL_NO_CONV_GAP")) {
      if (dycl_status s = dmalloc(g, &g->d_gap_part, part * 4)) return s;
      if (dycl_status s = dmalloc(g, &g->d_gap_pooled, pooled * 4)) return s;
    }
  }
  g->finalized = true;
  return DYCL_OK;
}

static dycl_status run_impl(dycl_graph g, const float* input, int64_t batch, float* logits, int32_t* path,
                            int32_t* node_counts, cudaStream_t st, long long global_offset = 0,
                            float* min_margin = nullptr, uint16_t* features = nullptr) {
  if (!g->finalized) return fail(g, DYCL_E_STATE, "graph not finalized");
  if (batch < 0 || batch > g->max_batch) return fail(g, DYCL_E_SHAPE_MISMATCH, "batch > max_batch");
  if (batch > 0 && (!input || !logits || !path)) return fail(g, DYCL_E_INVALID_ARG, "null io pointer");
  if (global_offset < 0) return fail(g, DYCL_E_INVALID_ARG, "negative global_offset");
  CK(cudaSetDevice(g->device));
  CK(cudaGetLastError());                      // surface async faults of earlier work
  g->prof_used = 0;
  g->prof_stream = st;
  g->rb_sent = g->rb_recv = 0;
  const bool rebal = g->tr && g->rb_policy != 0 && g->n_exits > 0;
  // a rebalanced run: lock step with the other ranks (even with no rows of its own: it may
  // receive some); results land in the library's result space first, then own rows go to the
  // caller. Device-initiated exchanges have no host step, so that run is graph-captured too.
  auto rebal_body = [&](cudaStream_t s, int* nlaunch) -> dycl_status {
    Exec ex{g, s, (int)std::max<int64_t>(batch, 1), g->d_res_logits, g->d_res_path};
    ex.out_margin = g->d_res_margin;
    ex.global_offset = global_offset;
    ex.own = (int)batch;
    if (dycl_status r = ex.run(input)) return r;
    *nlaunch = ex.nlaunch;
    if (batch > 0) {
      CK(cudaMemcpyAsync(logits, g->d_res_logits, (size_t)batch * g->K * 4, cudaMemcpyDeviceToDevice, s));
      CK(cudaMemcpyAsync(path, g->d_res_path, (size_t)batch * 4, cudaMemcpyDeviceToDevice, s));
      if (min_margin)
        CK(cudaMemcpyAsync(min_margin, g->d_res_margin, (size_t)batch * 4, cudaMemcpyDeviceToDevice, s));
    }
    return DYCL_OK;
  };
  const bool graphable = g->use_graph && !g->profiling && !g->dbg_ts && !features;
  if (rebal && g->rb_device && !g->drb_win) {
    // the symmetric window is set up collectively (every rank's first rebalanced run) -- before
    // any capture: its allocation / registration cannot be recorded into a graph
    std::string err;
    if (!g->tr->window(g->drb_bytes, &g->drb_win, &g->drb_peers, &err)) return fail(g, DYCL_E_NCCL, err);
  }
  if (rebal && !(g->rb_device && graphable)) {
    if (dycl_status r = rebal_body(st, &g->launches_per_run)) return r;
  } else if (batch == 0 && !rebal) {
    CK(cudaMemsetAsync(g->d_counts, 0, g->n_slots * sizeof(int), st));
  } else if (!rebal && !graphable) {
    Exec ex{g, st, (int)batch, logits, path};
    ex.out_margin = min_margin;
    ex.out_features = features;
    ex.own = (int)batch;
    if (dycl_status s = ex.run(input)) return s;
    g->launches_per_run = ex.nlaunch;
  } else {
    const void* key[4] = {input, logits, path, min_margin};
    const long long goff = rebal ? global_offset : -1;
    dycl_graph_s::GraphEntry* ge = nullptr;
    for (auto& e : g->graphs)
      if (e.exec && e.batch == batch && e.goff == goff && e.key[0] == key[0] && e.key[1] == key[1] &&
          e.key[2] == key[2] && e.key[3] == key[3])
        ge = &e;
    if (!ge) {
      ge = &g->graphs[0];                            // empty slot, else the least recently used
      for (auto& e : g->graphs)
        if (!e.exec || (ge->exec && e.used < ge->used)) ge = &e;
      if (ge->exec) {
        cudaGraphExecDestroy(ge->exec);
        ge->exec = nullptr;
      }
      if (!g->cap_stream) CK(cudaStreamCreateWithFlags(&g->cap_stream, cudaStreamNonBlocking));
      CK(cudaStreamBeginCapture(g->cap_stream, cudaStreamCaptureModeThreadLocal));
      int nl = 0;
      dycl_status r;
      if (rebal) {
        r = rebal_body(g->cap_stream, &nl);
      } else {
        Exec ex{g, g->cap_stream, (int)batch, logits, path};
        ex.out_margin = min_margin;
        ex.own = (int)batch;
        r = ex.run(input);
        nl = ex.nlaunch;
      }
      cudaGraph_t graph = nullptr;
      const cudaError_t ec = cudaStreamEndCapture(g->cap_stream, &graph);
      if (r != DYCL_OK) {
        if (graph) cudaGraphDestroy(graph);
        return r;
      }
      if (ec != cudaSuccess) return cuda_fail(g, ec, "graph capture");
      const cudaError_t ei = cudaGraphInstantiate(&ge->exec, graph, 0);
      cudaGraphDestroy(graph);
      if (ei != cudaSuccess) {
        ge->exec = nullptr;
        return cuda_fail(g, ei, "graph instantiate");
      }
      for (int i = 0; i < 4; ++i) ge->key[i] = key[i];
      ge->batch = batch;
      ge->goff = goff;
      ge->launches = nl;
    }
    ge->used = ++g->graph_clock;
    CK(cudaGraphLaunch(ge->exec, st));
    g->launches_per_run = ge->launches;
  }
  if (node_counts) CK(cudaMemcpyAsync(node_counts, g->d_counts, g->n_slots * sizeof(int), cudaMemcpyDeviceToDevice, st));
  return DYCL_OK;
}

dycl_status dycl_run(dycl_graph g, const dycl_io* io, void* stream) {
  if (!g || !io) return DYCL_E_INVALID_ARG;
  return run_impl(g, io->input, io->batch, io->logits, io->path, io->node_counts, (cudaStream_t)stream,
                  io->global_offset, io->min_margin, io->features);
}

static dycl_status run_host_impl(dycl_graph g, const float* input_host, int64_t batch, long long global_offset,
                                 float* logits_host, int32_t* path_host, float* margin_host, void* stream) {
  if (!g) return DYCL_E_INVALID_ARG;
  if (!g->finalized) return fail(g, DYCL_E_STATE, "graph not finalized");
  if (batch < 0) return fail(g, DYCL_E_SHAPE_MISMATCH, "negative batch");
  if (batch > 0 && (!input_host || !logits_host || !path_host)) return fail(g, DYCL_E_INVALID_ARG, "null pointer");
  CK(cudaSetDevice(g->device));
  cudaStream_t st = (cudaStream_t)stream;
  // a batch larger than the graph's max_batch streams through in max_batch-row sub-chunks, two
  // staging slots of max_batch rows each (only the first sub-chunk's copy is exposed)
  const bool big = batch > g->max_batch;
  const int64_t need = big ? 2 * g->max_batch : g->max_batch;
  if (g->stage_rows < need) {
    cudaFree(g->d_in_stage);
    cudaFree(g->d_logit_stage);
    cudaFree(g->d_path_stage);
    cudaFree(g->d_margin_stage);
    g->d_in_stage = nullptr; g->d_logit_stage = nullptr; g->d_path_stage = nullptr; g->d_margin_stage = nullptr;
    g->stage_rows = 0;
    const size_t in_elems = (size_t)need * g->input.H * g->input.W * g->input.C;
    if (dycl_status s = dmalloc(g, &g->d_in_stage, in_elems * 4)) return s;
    if (dycl_status s = dmalloc(g, &g->d_logit_stage, (size_t)need * g->K * 4)) return s;
    if (dycl_status s = dmalloc(g, &g->d_path_stage, (size_t)need * 4)) return s;
    if (dycl_status s = dmalloc(g, &g->d_margin_stage, (size_t)need * 4)) return s;
    g->stage_rows = need;
  }
  const size_t row_in = (size_t)g->input.H * g->input.W * g->input.C;
  // Pipelined over sub-chunks in two staging slots: H2D of sub-chunk k+1 (copy stream) and
  // D2H of k-1 (second copy stream) overlap the run of k on the caller's stream.  Samples are
  // independent and every kernel is batch-position independent, so the results equal one run.
  // sub-chunk: a quarter of the batch.  Small samples (< 64 KB of input), whose runs lose
  // efficiency below ~2048 rows: two uneven chunks, a quarter then the rest -- only the first
  // chunk's copy is exposed, the second one's hides under the first run
  int64_t sc = big ? g->max_batch : batch >= 1024 ? (batch + 3) / 4 : batch;
  int64_t first = sc;                              // rows of chunk 0
  const bool small = row_in * 4 < 64 * 1024 && !big;
  if (small) {
    if (batch >= 2048 && !getenv("DYCL_E2E_EVEN")) {
      first = ((batch + 3) / 4 + 255) / 256 * 256;
      sc = batch - first;                          // chunk 1 (slot 1 starts at row `first`)
    } else if (sc < 2048) {
      sc = first = std::min<int64_t>(batch, 2048);
    }
  }
  const bool uneven = small && first != sc && batch >= 2048 && first < batch;
  const int64_t nsc = batch <= 0 ? 0 : uneven ? 2 : (batch + sc - 1) / sc;
  if (nsc <= 1) {
    CK(cudaMemcpyAsync(g->d_in_stage, input_host, (size_t)batch * row_in * 4, cudaMemcpyHostToDevice, st));
    if (dycl_status s = run_impl(g, g->d_in_stage, batch, g->d_logit_stage, g->d_path_stage, nullptr, st,
                                 global_offset, margin_host ? g->d_margin_stage : nullptr))
      return s;
    CK(cudaMemcpyAsync(logits_host, g->d_logit_stage, (size_t)batch * g->K * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(path_host, g->d_path_stage, (size_t)batch * 4, cudaMemcpyDeviceToHost, st));
    if (margin_host)
      CK(cudaMemcpyAsync(margin_host, g->d_margin_stage, (size_t)batch * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return DYCL_OK;
  }
  if (!g->h2d_stream) {
    CK(cudaStreamCreateWithFlags(&g->h2d_stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&g->d2h_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      CK(cudaEventCreateWithFlags(&g->ev_h2d[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&g->ev_run[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&g->ev_d2h[i], cudaEventDisableTiming));
    }
  }
  for (int64_t k = 0; k < nsc; ++k) {
    const int slot = (int)(k & 1);
    const int64_t r0 = uneven ? (k == 0 ? 0 : first) : k * sc;
    const int64_t rows = uneven ? (k == 0 ? first : batch - first) : std::min<int64_t>(sc, batch - r0);
    const size_t off = uneven ? (size_t)r0 : (size_t)slot * sc;    // staging rows of this slot
    float* din = g->d_in_stage + off * row_in;
    float* dz = g->d_logit_stage + off * g->K;
    int32_t* dp = g->d_path_stage + off;
    float* dm = margin_host ? g->d_margin_stage + off : nullptr;
    if (k >= 2) CK(cudaStreamWaitEvent(g->h2d_stream, g->ev_run[slot], 0));     // run k-2 read this slot
    CK(cudaMemcpyAsync(din, input_host + (size_t)r0 * row_in, (size_t)rows * row_in * 4, cudaMemcpyHostToDevice,
                       g->h2d_stream));
    CK(cudaEventRecord(g->ev_h2d[slot], g->h2d_stream));
    CK(cudaStreamWaitEvent(st, g->ev_h2d[slot], 0));
    if (k >= 2) CK(cudaStreamWaitEvent(st, g->ev_d2h[slot], 0));                // D2H k-2 read this slot
    if (dycl_status s = run_impl(g, din, rows, dz, dp, nullptr, st, global_offset + r0, dm)) return s;
    CK(cudaEventRecord(g->ev_run[slot], st));
    CK(cudaStreamWaitEvent(g->d2h_stream, g->ev_run[slot], 0));
    CK(cudaMemcpyAsync(logits_host + (size_t)r0 * g->K, dz, (size_t)rows * g->K * 4, cudaMemcpyDeviceToHost,
                       g->d2h_stream));
    CK(cudaMemcpyAsync(path_host + r0, dp, (size_t)rows * 4, cudaMemcpyDeviceToHost, g->d2h_stream));
    if (margin_host) CK(cudaMemcpyAsync(margin_host + r0, dm, (size_t)rows * 4, cudaMemcpyDeviceToHost, g->d2h_stream));
    CK(cudaEventRecord(g->ev_d2h[slot], g->d2h_stream));
  }
  CK(cudaStreamSynchronize(g->d2h_stream));
  CK(cudaStreamSynchronize(st));
  return DYCL_OK;
}

dycl_status dycl_run_host(dycl_graph g, const float* input_host, int64_t batch, float* logits_host,
                          int32_t* path_host, void* stream) {
  return run_host_impl(g, input_host, batch, 0, logits_host, path_host, nullptr, stream);
}

dycl_status dycl_run_host_ex(dycl_graph g, const float* input_host, int64_t batch, int64_t global_offset,
                             float* logits_host, int32_t* path_host, float* min_margin_host, void* stream) {
  return run_host_impl(g, input_host, batch, global_offset, logits_host, path_host, min_margin_host, stream);
}

dycl_status dycl_num_count_slots(dycl_graph g, int32_t* out) {
  if (!g || !out) return DYCL_E_INVALID_ARG;
  if (!g->finalized) return fail(g, DYCL_E_STATE, "graph not finalized");
  *out = g->n_slots;
  return DYCL_OK;
}

dycl_status dycl_launches_per_run(dycl_graph g, int32_t* out) {
  if (!g || !out) return DYCL_E_INVALID_ARG;
  *out = g->launches_per_run;
  return DYCL_OK;
}

dycl_status dycl_num_classes(dycl_graph g, int32_t* out) {
  if (!g || !out) return DYCL_E_INVALID_ARG;
  if (!g->finalized) return fail(g, DYCL_E_STATE, "graph not finalized");
  *out = g->K;
  return DYCL_OK;
}

dycl_status dycl_set_profiling(dycl_graph g, int enable) {
  if (!g) return DYCL_E_INVALID_ARG;
  g->profiling = enable != 0;
  return DYCL_OK;
}

dycl_status dycl_profile_read(dycl_graph g, int32_t max_n, int32_t* kind, float* ms, double* bytes,
                              double* flops, int32_t* n_out) {
  if (!g || !n_out) return DYCL_E_INVALID_ARG;
  CK(cudaSetDevice(g->device));
  CK(cudaStreamSynchronize(g->prof_stream));
  std::vector<int> counts(g->n_slots, 0);
  if (g->d_counts) CK(cudaMemcpy(counts.data(), g->d_counts, g->n_slots * sizeof(int), cudaMemcpyDeviceToHost));
  const int n = (int)std::min<size_t>(g->prof_used, (size_t)std::max(max_n, 0));
  for (int i = 0; i < n; ++i) {
    const Launch& L = g->prof[i];
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, L.e0, L.e1));
    const double rows = L.count_dev ? (double)counts[L.count_dev - g->d_counts] : 0.0;
    if (kind) kind[i] = L.kind;
    if (ms) ms[i] = t;
    if (bytes) bytes[i] = rows * L.bytes_per_row + L.bytes_fixed;
    if (flops) flops[i] = rows * L.flops_per_row;
  }
  *n_out = (int32_t)g->prof_used;
  return DYCL_OK;
}

dycl_status dycl_debug_conv2d(dycl_graph g, int64_t n, int H, int W, int C, const uint16_t* w, const float* bias,
                              int c_out, int k, int stride, int pad, int relu, const void* res, int res_mode,
                              const void* x, void* y, int path) {
  if (!g || !w || !bias || !x || !y || n < 0 || C % 8 || c_out % 16 || k < 1 || stride < 1 || res_mode < 0 ||
      res_mode > 2 || (res_mode && !res))
    return fail(g, DYCL_E_INVALID_ARG, "debug_conv2d: bad argument");
  CK(cudaSetDevice(g->device));
  const int Ho = (H + 2 * pad - k) / stride + 1, Wo = (W + 2 * pad - k) / stride + 1;
  const int K = k * k * C, Kp = (K + 63) / 64 * 64;
  std::vector<uint16_t> wp((size_t)c_out * Kp, 0);
  for (int o = 0; o < c_out; ++o)
    for (int j = 0; j < K; ++j) wp[(size_t)o * Kp + j] = w[(size_t)o * K + j];
  uint16_t* dw = nullptr;
  float* db = nullptr;
  if (dycl_status s = dmalloc(g, &dw, wp.size() * 2)) return s;
  if (dycl_status s = dmalloc(g, &db, (size_t)c_out * 4)) { cudaFree(dw); return s; }
  cudaMemcpy(dw, wp.data(), wp.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, bias, (size_t)c_out * 4, cudaMemcpyHostToDevice);
  uint16_t* dwr = nullptr;
  int kp_rt = 0;
  if (k == 3 && stride == 1 && pad == 1 && path != 3 && path != 4) {   // (path 5 included)
    kp_rt = (3 * C + 63) / 64 * 64;
    std::vector<uint16_t> wr((size_t)3 * c_out * kp_rt);
    dycl::pack_rowtap(wp.data(), c_out, Kp, C, wr.data(), kp_rt);
    if (cudaMalloc(&dwr, wr.size() * 2) == cudaSuccess) cudaMemcpy(dwr, wr.data(), wr.size() * 2, cudaMemcpyHostToDevice);
  }
  dycl::ConvArgs a{};
  a.x = (const uint16_t*)x; a.w = dw; a.w_rt = dwr; a.Kp_rt = kp_rt; a.bias = db;
  a.res = (const uint16_t*)res; a.y = (uint16_t*)y;
  a.n_live = nullptr; a.n_static = (int)n;
  a.H = H; a.W = W; a.C = C; a.Ho = Ho; a.Wo = Wo; a.Cout = c_out; a.ksz = k; a.stride = stride; a.pad = pad;
  a.K = K; a.Kp = Kp; a.relu = relu; a.res_mode = res_mode;
  a.rH = 2 * Ho; a.rW = 2 * Wo; a.rC = c_out / 2; a.r_pad_lo = c_out / 4;
  if (res_mode == 1) { a.rH = Ho; a.rW = Wo; a.rC = c_out; a.r_pad_lo = 0; }
  if (path == 2 && dwr) a.dbg |= 32;          // path 2 exercises the row-tap mode where eligible
  // path 4: NHWC tensors, im2col GEMM (8-channel stem: planar kernels); 5: the same with row-tap
  // weights supplied (the GEMM's row-tap form where eligible)
  a.nhwc = a.in_nhwc = a.res_nhwc = path == 4 || path == 5;
  cudaError_t e = n > 0 ? dycl::launch_conv(a, (int)n, g->num_sms, 0, path == 3 ? 2 : path >= 4 ? 0 : path)
                        : cudaSuccess;
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  cudaFree(dwr);
  cudaFree(dw);
  cudaFree(db);
  if (e != cudaSuccess) return cuda_fail(g, e, "debug_conv2d");
  return DYCL_OK;
}

// Result space + exchange staging for rebalancing runs (allocated when a transport is set).
static dycl_status alloc_rebalance(dycl_graph g) {
  const int levels = std::max(1, std::min(g->n_exits, 31));
  const int64_t rows = (int64_t)g->max_batch * (1 + levels);
  const size_t K = (size_t)std::max(g->K, 1), mb = (size_t)g->max_batch;
  dycl_status s;
  if ((s = dmalloc(g, &g->d_res_logits, (size_t)rows * K * 4)) || (s = dmalloc(g, &g->d_res_path, rows * 4)) ||
      (s = dmalloc(g, &g->d_res_margin, rows * 4)) || (s = dmalloc(g, &g->d_ext_gid, rows * 8)) ||
      (s = dmalloc(g, &g->d_sent_orig, rows * 4)) || (s = dmalloc(g, &g->d_meta, 2 * mb * 16)) ||
      (s = dmalloc(g, &g->d_ret_logits, (size_t)rows * K * 4)) || (s = dmalloc(g, &g->d_ret_path, rows * 4)) ||
      (s = dmalloc(g, &g->d_ret_margin, rows * 4)))
    return s;
  g->rb_rows = rows;
  return DYCL_OK;
}

static dycl_status set_transport(dycl_graph g, dycl::Transport* t, int policy) {
  CK(cudaSetDevice(g->device));
  delete g->tr;
  g->tr = t;
  g->rb_policy = policy;
  if (t && policy != 0 && !g->d_res_logits) return alloc_rebalance(g);
  return DYCL_OK;
}

dycl_status dycl_set_comm(dycl_graph g, void* nccl_comm, int rank, int world, int rebalance_policy) {
  if (!g) return DYCL_E_INVALID_ARG;
  if (!g->finalized) return fail(g, DYCL_E_STATE, "dycl_set_comm: finalize the graph first");
  if (world < 1 || rank < 0 || rank >= world || (world > 1 && !nccl_comm))
    return fail(g, DYCL_E_INVALID_ARG, "dycl_set_comm: bad rank / world / communicator");
  if (world == 1 && !nccl_comm) return set_transport(g, nullptr, 0);
  std::string err;
  dycl::Transport* t = dycl::make_nccl_transport(nccl_comm, rank, world, &err);
  if (!t) return fail(g, DYCL_E_NCCL, err);
  return set_transport(g, t, rebalance_policy);
}

// dycl::preload_kernels, tolerating a driver without the module-enumeration entry points (the
// preload only removes a lazy-loading stall between in-process ranks; it is not needed for
// correctness of a single-rank or multi-process run)
static cudaError_t preload_or_skip() {
  const cudaError_t e = dycl::preload_kernels();
  return e == cudaErrorNotSupported ? cudaSuccess : e;
}

dycl_status dycl_set_rebalance_mode(dycl_graph g, int mode) {
  if (!g) return DYCL_E_INVALID_ARG;
  if (mode != DYCL_REBALANCE_MODE_HOST && mode != DYCL_REBALANCE_MODE_DEVICE)
    return fail(g, DYCL_E_INVALID_ARG, "rebalance mode");
  if (!g->tr || !g->d_res_logits) return fail(g, DYCL_E_STATE, "dycl_set_rebalance_mode: attach a communicator first");
  if (mode == DYCL_REBALANCE_MODE_DEVICE && g->tr->world > dycl::DRB_MAX_WORLD)
    return fail(g, DYCL_E_UNSUPPORTED, "device rebalancing: at most 8 ranks (one NVLink domain)");
  CK(cudaSetDevice(g->device));
  g->rb_device = mode == DYCL_REBALANCE_MODE_DEVICE;
  // every kernel loaded before the first exchange: a lazy load during a run could wait for a
  // context that one of this process's spinning exchange kernels keeps busy (kernels.h)
  if (g->rb_device) CK(preload_or_skip());
  if (g->rb_device && !g->d_drb_plan) {
    dycl_status s;
    if ((s = dmalloc(g, &g->d_drb_plan, dycl::DRB_MAX_LEVELS * sizeof(dycl::DrbPlan))) ||
        (s = dmalloc(g, &g->d_drb_epoch, sizeof(unsigned))) || (s = dmalloc(g, &g->d_drb_err, sizeof(int))) ||
        (s = dmalloc(g, &g->d_drb_ticket, sizeof(int))))
      return s;
    CK(cudaMemset(g->d_drb_plan, 0, dycl::DRB_MAX_LEVELS * sizeof(dycl::DrbPlan)));
    CK(cudaMemset(g->d_drb_epoch, 0, sizeof(unsigned)));
    CK(cudaMemset(g->d_drb_err, 0, sizeof(int)));
    CK(cudaMemset(g->d_drb_ticket, 0, sizeof(int)));
    // window: control words | max_batch row slots (the largest exit input: bf16 + fp32 planes +
    // 16 B) | per level max_batch returned results (K logits, path, margin, pad)
    long long row = 16;
    for (const Node& N : g->nodes)
      if (N.kind == N_EXIT) row = std::max(row, N.in.row_elems() * 6 + 16);
    const size_t ctrl = (sizeof(dycl::DrbCtrl) + 255) / 256 * 256;
    const size_t rows = ((size_t)g->max_batch * row + 255) / 256 * 256;
    const size_t levels = (size_t)std::max(1, std::min(g->n_exits, dycl::DRB_MAX_LEVELS));
    const size_t ret = levels * (size_t)g->max_batch * ((size_t)g->K + 4) * 4;
    g->drb_rows_off = ctrl;
    g->drb_ret_off = ctrl + rows;
    g->drb_bytes = (ctrl + rows + ret + 4095) / 4096 * 4096;
  }
  return DYCL_OK;
}

struct dycl_local_group_s {
  dycl::LocalGroup* g;
};

dycl_status dycl_local_group_create(int world, dycl_local_group* out) {
  if (world < 1 || !out) return fail(nullptr, DYCL_E_INVALID_ARG, "bad world");
  *out = new (std::nothrow) dycl_local_group_s{dycl::local_group_create(world)};
  return *out ? DYCL_OK : DYCL_E_OOM;
}

dycl_status dycl_local_group_destroy(dycl_local_group grp) {
  if (grp) {
    dycl::local_group_destroy(grp->g);
    delete grp;
  }
  return DYCL_OK;
}

dycl_status dycl_set_comm_local(dycl_graph g, dycl_local_group grp, int rank, int rebalance_policy) {
  if (!g || !grp) return DYCL_E_INVALID_ARG;
  if (!g->finalized) return fail(g, DYCL_E_STATE, "dycl_set_comm_local: finalize the graph first");
  const int world = dycl::local_group_world(grp->g);
  if (rank < 0 || rank >= world) return fail(g, DYCL_E_INVALID_ARG, "bad rank");
  // in-process ranks share one GPU: with device-initiated rebalancing a rank's wait kernels spin
  // on an SM while the others compute, so compute grids leave `world` SMs free (a persistent
  // grid of one CTA per SM could otherwise never start its last CTA behind a spinner)
  if (world > 1 && g->num_sms > world) g->num_sms -= world;
  CK(cudaSetDevice(g->device));
  CK(preload_or_skip());                       // ranks of one process share one context (kernels.h)
  return set_transport(g, dycl::make_local_transport(grp->g, rank), rebalance_policy);
}

dycl_status dycl_rebalance_stats(dycl_graph g, int64_t* rows_sent, int64_t* rows_received) {
  if (!g || !rows_sent || !rows_received) return DYCL_E_INVALID_ARG;
  if (g->rb_device && g->d_drb_plan) {
    // the plans live on the device: read the last run's levels (and its error word)
    CK(cudaSetDevice(g->device));
    CK(cudaDeviceSynchronize());
    int err = 0;
    CK(cudaMemcpy(&err, g->d_drb_err, sizeof(int), cudaMemcpyDeviceToHost));
    if (err) return fail(g, DYCL_E_NCCL, "device rebalancing: " +
                                             std::string(err == 2 ? "rows held exceed max_batch" : "peer wait timed out"));
    std::vector<dycl::DrbPlan> P(dycl::DRB_MAX_LEVELS);
    CK(cudaMemcpy(P.data(), g->d_drb_plan, P.size() * sizeof(dycl::DrbPlan), cudaMemcpyDeviceToHost));
    long long sent = 0, recv = 0;
    for (int k = 0; k < g->drb_levels_last; ++k) {
      sent += P[k].n_send;
      recv += P[k].n_recv;
    }
    *rows_sent = sent;
    *rows_received = recv;
    return DYCL_OK;
  }
  *rows_sent = g->rb_sent;
  *rows_received = g->rb_recv;
  return DYCL_OK;
}

dycl_status dycl_nccl_get_unique_id(uint8_t out[128]) {
  if (!out) return fail(nullptr, DYCL_E_INVALID_ARG, "null");
  std::string err;
  if (!dycl::nccl_get_unique_id(out, &err)) return fail(nullptr, DYCL_E_NCCL, err);
  return DYCL_OK;
}

dycl_status dycl_nccl_comm_init_rank(const uint8_t id[128], int rank, int world, int cuda_device, void** comm) {
  if (!id || !comm || world < 1 || rank < 0 || rank >= world) return fail(nullptr, DYCL_E_INVALID_ARG, "bad argument");
  if (cudaSetDevice(cuda_device) != cudaSuccess) return fail(nullptr, DYCL_E_CUDA, "cudaSetDevice");
  std::string err;
  if (!dycl::nccl_comm_init_rank(id, rank, world, comm, &err)) return fail(nullptr, DYCL_E_NCCL, err);
  return DYCL_OK;
}

dycl_status dycl_nccl_comm_destroy(void* comm) {
  if (!comm) return DYCL_OK;
  std::string err;
  if (!dycl::nccl_comm_destroy(comm, &err)) return fail(nullptr, DYCL_E_NCCL, err);
  return DYCL_OK;
}

dycl_status dycl_rebalance_plan(const int32_t* counts, int world, int rank, int32_t* send, int32_t* recv,
                                int32_t* new_count) {
  if (!counts || world < 1 || rank < 0 || rank >= world || !send || !recv || !new_count)
    return fail(nullptr, DYCL_E_INVALID_ARG, "rebalance_plan: bad argument");
  long long S = 0;
  for (int r = 0; r < world; ++r) {
    if (counts[r] < 0) return fail(nullptr, DYCL_E_INVALID_ARG, "rebalance_plan: negative count");
    S += counts[r];
  }
  const long long T = (S + world - 1) / world;
  for (int j = 0; j < world; ++j) send[j] = recv[j] = 0;
  // two-pointer matching: surplus ranks (ascending) give to deficit ranks (ascending)
  std::vector<long long> give(world), take(world);
  for (int r = 0; r < world; ++r) {
    give[r] = counts[r] > T ? counts[r] - T : 0;
    take[r] = counts[r] < T ? T - counts[r] : 0;
  }
  int d = 0;
  for (int sr = 0; sr < world; ++sr) {
    while (give[sr] > 0) {
      while (d < world && take[d] == 0) ++d;
      if (d >= world) break;                 // cannot happen: total deficit >= total surplus
      const long long m = give[sr] < take[d] ? give[sr] : take[d];
      if (sr == rank) send[d] += (int32_t)m;
      if (d == rank) recv[sr] += (int32_t)m;
      give[sr] -= m;
      take[d] -= m;
    }
  }
  long long held = counts[rank];
  for (int j = 0; j < world; ++j) held += recv[j] - send[j];
  *new_count = (int32_t)held;
  return DYCL_OK;
}

dycl_status dycl_debug_timestamps(dycl_graph g, long long* out128) {
  if (!g || !out128) return DYCL_E_INVALID_ARG;
  if (!g->dbg_ts) return fail(g, DYCL_E_STATE, "DYCL_TS not set");
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(out128, g->dbg_ts, 128 * sizeof(long long), cudaMemcpyDeviceToHost));
  return DYCL_OK;
}

}  // extern "C"
