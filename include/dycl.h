/*
 * dycl.h -- C ABI of libdycl.so: batched inference of a dynamic neural network
 * (DyNN) that has been rewritten into conditional-free sub-networks plus a host
 * module holding the control flow (DyCL, arXiv 2307.04963), executed on B200.
 *
 * The paper's problem statement (Sec. 5 Eq. 2): given a DyNN
 * P_DyNN, produce a host program P_Host with P_DyNN(x) = P_Host(x) for all x.
 * P_Host "invokes" compiled sub-DNNs and holds the conditionals (PAPER.md
 * L534-535, L720); the deployment verbs are set_input / run / get_output
 * (Listing 2).  This library is the run-time half of that picture:
 *
 *   - sub-networks (HCFG tensor nodes, Sec. 5.3) are registered layer
 *     by layer; each runs as sm_100a tcgen05 kernels over the samples that take it;
 *   - logic nodes (HCFG logic nodes: exit, gate, final) are registered in program
 *     order as a chain; their predicates run per sample on the device;
 *   - the host module itself (branching, compaction of the rows that take each
 *     branch, scatter of results to the original order) runs on the device, so a
 *     run has NO host round trip.
 *
 * Conventions (apply to every function):
 *   - Return value: dycl_status; 0 == DYCL_OK, negative values are errors.  No C++
 *     exception crosses this ABI and nothing aborts the process.
 *   - On error, dycl_last_error(g) returns a human-readable message.
 *   - Host pointers passed at registration are COPIED before the call returns
 *     (weight snapshot semantics); the caller may free them.
 *   - Device pointers passed to dycl_run are caller-owned and must stay valid until
 *     the work enqueued on `stream` completes.  The library owns its workspace
 *     (allocated in dycl_finalize, freed in dycl_graph_destroy).
 *   - A graph is immutable after dycl_finalize; one dycl_run in
 *     flight per graph; use one graph per stream for concurrency.
 *   - Layouts: per-sample activations are NHWC ([H][W][C], C fastest); bf16 values
 *     are passed as their uint16 bit patterns.
 */
#ifndef DYCL_H_
#define DYCL_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dycl_graph_s* dycl_graph;
typedef int32_t dycl_node;      /* sub-network id, assigned in creation order from 0 */

typedef enum {
  DYCL_OK = 0,
  DYCL_E_INVALID_ARG = -1,      /* null pointer, out-of-range value                     */
  DYCL_E_SHAPE_MISMATCH = -2,   /* layer shape rule violated, batch > max */
  DYCL_E_SIGNATURE = -3,        /* head output widths disagree                          */
  DYCL_E_SHAPE_JOIN = -4,       /* gate then-branch vs skip output shapes*/
  DYCL_E_STATE = -5,            /* call not allowed in this state (finalized / not)     */
  DYCL_E_UNSUPPORTED = -6,      /* valid request this build does not implement          */
  DYCL_E_OOM = -7,              /* device allocation failed                             */
  DYCL_E_CUDA = -8,             /* CUDA runtime error (text in dycl_last_error)         */
  DYCL_E_NCCL = -9
} dycl_status;

typedef enum { DYCL_ACT_NONE = 0, DYCL_ACT_RELU = 1 } dycl_act;

/* ---------------------------------------------------------------- graphs --- */

/* Create an empty graph on CUDA device `cuda_device` whose per-sample input is an
 * fp32 NHWC tensor [in_h][in_w][in_c] (an MLP input of width d is [1][1][d]).
 * The run's first step (a0, Listing 2's pre-processing) casts
 * it to bf16 and pads channels to a multiple of 8.  *out receives the handle. */
dycl_status dycl_graph_create(int cuda_device, int in_h, int in_w, int in_c, dycl_graph* out);

/* Numerics of the activations between layers (call before dycl_finalize).
 * Tensor-core operands are always bf16 with fp32 accumulation.
 *   DYCL_PREC_FP32_STREAM (default): residual-stream tensors (block inputs/outputs,
 *     sub-network outputs) are kept in fp32; each conv/dense reads a bf16 (RNE)
 *     copy of its input; intermediates inside a block are bf16.
 *   DYCL_PREC_BF16: every activation is stored bf16 (half the bytes; logits drift
 *     ~4e-2 relative after 27 blocks, past the 2e-2 bar -- see DESIGN.md §2 reading R13).
 *   DYCL_PREC_BF16X3_PARITY: DYCL_E_UNSUPPORTED for image graphs (implemented for the
 *     generative graph, dycl_s2s_set_precision; image graphs show 0 outside-band decision
 *     mismatches in FP32_STREAM on 512 / 512 / 256 oracle samples, R13). */
enum { DYCL_PREC_BF16 = 0, DYCL_PREC_FP32_STREAM = 1, DYCL_PREC_BF16X3_PARITY = 2 };
dycl_status dycl_graph_set_precision(dycl_graph g, int precision);

/* Free the graph and all device memory it owns.  NULL is accepted. */
dycl_status dycl_graph_destroy(dycl_graph g);

/* Last error message for g (or for failed dycl_graph_create if g == NULL).
 * Library-owned; valid until the next call on g. Never NULL. */
const char* dycl_last_error(dycl_graph g);

/* ------------------------------------------------------- sub-networks ------ */
/* A sub-network is a conditional-free straight-line layer list (an HCFG tensor
 * node).  Its input shape is the shape flowing into the logic
 * node that uses it; shapes are propagated at dycl_finalize exactly as Alg. 2
 * propagates them: a logic node's output shape is its
 * predecessor's, a tensor node is compiled for its predecessor's output shape. */

dycl_status dycl_subnet_begin(dycl_graph g, dycl_node* out);

/* Mark the current tensor as the shortcut source of a residual block. */
dycl_status dycl_subnet_block_begin(dycl_graph g, dycl_node sn);

/* 2-D convolution (the 'convolutional operator'):
 *   y[ho][wo][o] = act( b[o] + sum_{r,s,c} w[o][r][s][c] x[ho*stride-pad+r][wo*stride-pad+s][c]
 *                       (+ shortcut[ho][wo][o] if residual) )
 * w: host bf16 bits [c_out][k][k][c_in]; b: host fp32 [c_out].  c_in must equal
 * the channel count that shape propagation delivers to this layer (checked at
 * dycl_finalize, DYCL_E_SHAPE_MISMATCH otherwise); it sizes the weight snapshot.  residual = 1 adds the tensor saved by the last
 * dycl_subnet_block_begin: as is when its shape equals the output's, or the
 * parameter-free 'option A' shortcut (stride-2 subsample, (c_out-c_in)/2 zero
 * channels each side) when the output halves H, W and doubles C.  Else
 * DYCL_E_SHAPE_MISMATCH (reported at dycl_finalize).  c_out % 16 == 0 (tensor-core
 * N granularity), 1 <= k <= 7, stride in {1, 2}. */
dycl_status dycl_subnet_conv2d(dycl_graph g, dycl_node sn, int c_in, int c_out, int k, int stride, int pad,
                               const uint16_t* w_bf16, const float* bias, dycl_act act, int residual);

/* Dense layer (the 'dense operator') on a [1][1][n_in] tensor:
 * y = act(W x + b), W: host bf16 bits [n_out][n_in], b: host fp32 [n_out]
 * (n_in checked at dycl_finalize like conv2d's c_in).
 * If out_fp32 == 0 the layer runs on tensor cores and stores bf16 (n_out % 16 == 0).
 * If out_fp32 == 1 the layer is a classifier / gate head producing fp32 logits
 * (any n_out >= 1); it must be the last layer of its sub-network. */
dycl_status dycl_subnet_dense(dycl_graph g, dycl_node sn, int n_in, int n_out, const uint16_t* w_bf16,
                              const float* bias, dycl_act act, int out_fp32);

/* Projection shortcut (ResNet "option B"): a 1x1 convolution with the given stride
 * applied to the tensor saved by dycl_subnet_block_begin; its output (c_out channels,
 * no activation) replaces the saved tensor as the shortcut the next residual conv adds.
 * w: host bf16 [c_out][1][1][c_in], b: host fp32 [c_out]; c_in = the saved tensor's
 * channel count (checked at dycl_finalize). */
dycl_status dycl_subnet_projection(dycl_graph g, dycl_node sn, int c_in, int c_out, int stride,
                                   const uint16_t* w_bf16, const float* bias);

/* Max pooling with a k x k window, stride, zero-size padding of `pad` pixels on each side
 * (padded positions never win): y[ho][wo][c] = max over the window (torchvision MaxPool2d). */
dycl_status dycl_subnet_maxpool(dycl_graph g, dycl_node sn, int k, int stride, int pad);

/* Global average pooling [H][W][C] -> [1][1][C], fp32 mean (kept in fp32 when
 * followed by an out_fp32 dense head). */
dycl_status dycl_subnet_gap(dycl_graph g, dycl_node sn);

dycl_status dycl_subnet_end(dycl_graph g, dycl_node sn);

/* ---------------------------------------------------------- logic nodes ---- */
/* Registered in program order; together they form the host module.  Each uses
 * the current per-sample tensor h of the samples still running. */

/* h <- subnet(h) for every live sample. */
dycl_status dycl_seq(dycl_graph g, dycl_node subnet);

/* Early exit (Shallow-Deep): z = head(h) (fp32 logits [K]);
 * samples with max_j softmax(z)_j >= tau terminate: their logits z and
 * path = (index of this exit among the graph's exits) are written to the
 * outputs at their ORIGINAL batch position; the others continue with h. */
dycl_status dycl_exit(dycl_graph g, dycl_node head_subnet, float tau);

/* Conditional skip (SkipNet, Listing 3): z = gate(h) (one fp32
 * logit); samples with sigmoid(z) > thr run h <- then_subnet(h) and set bit
 * (index of this gate) in their path word; the others take the skip path
 * (identity, or option A when then_subnet halves H, W and doubles C -- the only
 * two join shapes accepted, else DYCL_E_SHAPE_JOIN). */
dycl_status dycl_gate(dycl_graph g, dycl_node gate_subnet, float thr, dycl_node then_subnet);

/* Recurrent conditional skip (SkipNet's RNN gate: Table 3 ID 5 "ResNet38 + RNN", PAPER.md L812;
 * Table 1).  One LSTM cell per graph, shared by every dycl_gate_rnn node and carrying a
 * per-sample state (h, c) across the gates in program order (zero at the start of a run):
 *   dycl_rnn_cell: hidden H <= 16, input width n_in <= 16; fp32 host weights (copied)
 *     w_ih [4H][n_in], w_hh [4H][H], b_ih [4H], b_hh [4H], gate rows in the order i, f, g, o
 *     (torch.nn.LSTMCell): (i,f,g,o) = (sig, sig, tanh, sig)(w_ih u + b_ih + w_hh h + b_hh);
 *     c <- f*c + i*g;  h <- o*tanh(c).
 *   dycl_gate_rnn: u = proj_subnet(h_act) (fp32 [n_in], e.g. GAP + dense(out_fp32)); the cell
 *     steps on u; z = w_out . h + b_out (w_out fp32 [H], copied); samples with sigmoid(z) > thr
 *     run then_subnet and set their path bit, as dycl_gate.  The cell steps for EVERY live sample
 *     at every gate, executed or not (the gate reads the block input).
 * Errors: dycl_rnn_cell twice or after a dycl_gate_rnn -> STATE; dycl_gate_rnn before
 * dycl_rnn_cell -> STATE; sizes out of range -> INVALID_ARG; proj_subnet output width != n_in
 * -> SHAPE_MISMATCH (at dycl_finalize).  A graph with recurrent gates never rebalances. */
dycl_status dycl_rnn_cell(dycl_graph g, int n_in, int hidden, const float* w_ih, const float* w_hh,
                          const float* b_ih, const float* b_hh);
dycl_status dycl_gate_rnn(dycl_graph g, dycl_node proj_subnet, const float* w_out, float b_out, float thr,
                          dycl_node then_subnet);

/* Default exit: every sample still running terminates with z = head(h).
 * path = number of exits registered (early-exit nets) or the gate mask. */
dycl_status dycl_final(dycl_graph g, dycl_node head_subnet);

/* Alg. 2 analog: shape propagation over the chain, buffer planning for
 * max_batch samples, weight upload to HBM.  Errors: SHAPE_MISMATCH, SHAPE_JOIN,
 * SIGNATURE, OOM, CUDA. */
dycl_status dycl_finalize(dycl_graph g, int64_t max_batch);

/* ------------------------------------------------------------------ run ---- */
typedef struct {
  const float* input;     /* device fp32 [batch][in_h][in_w][in_c] (NHWC)             */
  int64_t batch;          /* 0 <= batch <= max_batch                                  */
  float* logits;          /* device fp32 [batch][K]   (output, original order)        */
  int32_t* path;          /* device int32 [batch]     exit index or gate mask word     */
  int32_t* node_counts;   /* device int32 [dycl_num_count_slots] live-row counts, or NULL */
  int64_t global_offset;  /* global index of row 0 when the batch is one shard of a larger one
                             (rank r holds [r*B/G, (r+1)*B/G)); rows handed to other
                             ranks by rebalancing carry global_offset + row as their id.  >= 0.  */
  float* min_margin;      /* device fp32 [batch] or NULL: per sample, the minimum over the exit /
                             gate predicates evaluated along its path of |p - threshold| (p = max
                             softmax for exits, sigmoid for gates; +inf if none) -- the quantity the
                             north star's "within 1e-3 of its threshold" band is defined on (R12) */
  uint16_t* features;     /* device bf16 [batch][H][W][C] (NHWC) or NULL: the tensor entering the final
                             head, in input order -- the encoder output of an En-Decoder
                             (dycl_cap_run).  Plain graphs only (no exit / gate nodes) whose final
                             tensor is NHWC (C % 64 == 0); else DYCL_E_UNSUPPORTED */
} dycl_io;

/* Enqueue one batched inference on `stream` (a cudaStream_t, NULL = default stream).
 * Asynchronous and stream-ordered; no host synchronisation and no device->host
 * traffic.  Output row i always belongs to input row i. */
dycl_status dycl_run(dycl_graph g, const dycl_io* io, void* stream);

/* Same, with HOST buffers (pinned or pageable): copies the input host->device,
 * runs, copies logits and path device->host, and synchronises `stream` before
 * returning -- the deployment-style call of Listing 2 (set_input/run/get_output).
 * Any batch >= 0 is accepted: a batch larger than max_batch streams through in
 * max_batch-row sub-chunks (library-owned staging of 2 x max_batch rows).
 * Batches of >= 1024 rows are pipelined in sub-chunks (a quarter of the batch; for samples
 * under 64 KB, batches of >= 2048 rows run as two chunks, a quarter then the rest, so only
 * the first chunk's copy is exposed) over two library-owned
 * staging slots: the host->device copy of sub-chunk k+1 and the device->host copy of
 * k-1 run on two internal copy streams while sub-chunk k runs on `stream` (results
 * equal one run: samples are independent). */
dycl_status dycl_run_host(dycl_graph g, const float* input_host, int64_t batch,
                          float* logits_host, int32_t* path_host, void* stream);
/* dycl_run_host with the dycl_io extensions: global_offset (a shard of a global batch; every
 * sub-chunk run carries global_offset + its first row) and an optional host min_margin [batch]. */
dycl_status dycl_run_host_ex(dycl_graph g, const float* input_host, int64_t batch, int64_t global_offset,
                             float* logits_host, int32_t* path_host, float* min_margin_host, void* stream);

/* --------------------------------------------------------- introspection --- */
/* Number of device count slots a run writes (for dycl_io.node_counts). */
dycl_status dycl_num_count_slots(dycl_graph g, int32_t* out);
/* Number of this library's kernels one dycl_run launches. */
dycl_status dycl_launches_per_run(dycl_graph g, int32_t* out);
/* Output width K of the heads (valid after finalize). */
dycl_status dycl_num_classes(dycl_graph g, int32_t* out);

/* Per-launch profiling: when enabled, dycl_run brackets every launch with CUDA
 * events on the run's stream.  dycl_profile_read synchronises the last run's
 * stream and returns, per launch in issue order: kind (see DYCL_K_*), elapsed ms,
 * and the launch's algorithmic bytes and flops (computed from the live-row counts
 * the launch processed, read back AFTER the run).  Arrays hold max_n entries;
 * *n_out receives the number of launches. */
enum { DYCL_K_INPUT = 0, DYCL_K_CONV = 1, DYCL_K_HEAD = 2, DYCL_K_COMPACT = 3,
       DYCL_K_GATHER = 4, DYCL_K_SCATTER = 5, DYCL_K_INIT = 6, DYCL_K_POOL = 7,
       DYCL_K_BLOCK = 8 /* fused residual blocks (k_block_fused) */, DYCL_K_GEMM = 9 /* dense GEMM */,
       DYCL_K_ATTN = 10, DYCL_K_LN = 11, DYCL_K_ARGMAX = 12, DYCL_K_EMBED = 13 };
dycl_status dycl_set_profiling(dycl_graph g, int enable);
dycl_status dycl_profile_read(dycl_graph g, int32_t max_n, int32_t* kind, float* ms,
                              double* bytes, double* flops, int32_t* n_out);

/* ------------------------------------------------- multi-GPU rebalancing ---- */
/* Samples are independent (Eq. 2 is per x), so a global batch shards across
 * ranks with no collective: each rank runs its contiguous slice with dycl_io.global_offset.
 * Optional survivor rebalancing: after the exits selected by the policy, the
 * ranks all-gather their survivor counts (one int32 each; the run's one host synchronisation
 * per rebalanced exit), every rank computes the same plan (dycl_rebalance_plan below), and
 * surplus rows -- the bf16 / fp32 activation rows the next sub-network reads, plus 16 bytes of
 * metadata (path word, min margin, 64-bit global id) -- move in one grouped point-to-point step
 * on the run's stream.  Received rows are appended after the local survivors and run through
 * the rest of the chain with them.  At the end the results of rows computed away from home go
 * back by the reverse plans (last level first) and are scattered to their original rows by a
 * kernel.  Every kernel is batch-position independent, so the outputs are bitwise those of the
 * unbalanced run (tested).  A rebalancing run is issued launch by launch (no CUDA graph: it
 * reads the counts on the host); all ranks must call dycl_run the same number of times (lock
 * step), each with its own shard (batch may be 0).
 *
 * Policy: bit k set = rebalance after exit k; DYCL_REBALANCE_ALL = every exit; 0 = none
 * (shards only).  Graphs without exits (gates only) never rebalance. */
enum { DYCL_REBALANCE_NONE = 0, DYCL_REBALANCE_ALL = -1 };
/* nccl_comm: an ncclComm_t spanning the `world` ranks, this process being `rank` (borrowed, not
 * destroyed; e.g. torch's ProcessGroupNCCL._comm_ptr(), or dycl_nccl_comm_init_rank).  NCCL is
 * resolved at run time from the libnccl.so.2 mapped in the process.  nccl_comm == NULL with
 * world == 1 detaches (a world-1 communicator is kept: its runs all-gather and never move rows).
 * Call after dycl_finalize (allocates the result space: (1 + #exits) x max_batch rows).
 * Errors: INVALID_ARG, STATE, NCCL (library not found), OOM.  Run-time transport failures
 * surface from dycl_run as DYCL_E_NCCL. */
dycl_status dycl_set_comm(dycl_graph g, void* nccl_comm, int rank, int world, int rebalance_policy);
/* In-process transport: `world` graphs of one process (same or different devices), each driven
 * by its own host thread, exchange rows by device-to-device copies behind a host barrier.  Same
 * protocol and plan as the NCCL transport; used to test rebalancing on a single GPU. */
typedef struct dycl_local_group_s* dycl_local_group;
dycl_status dycl_local_group_create(int world, dycl_local_group* out);
dycl_status dycl_local_group_destroy(dycl_local_group grp);
dycl_status dycl_set_comm_local(dycl_graph g, dycl_local_group grp, int rank, int rebalance_policy);
/* Where the exchange runs (call after dycl_set_comm / dycl_set_comm_local; default HOST):
 *   DYCL_REBALANCE_MODE_HOST   as described above: count all-gather read on the host, host plan,
 *                              grouped point-to-point step (NCCL send / recv or local copies);
 *   DYCL_REBALANCE_MODE_DEVICE device-initiated: every rank owns a symmetric device
 *                              window (NCCL: ncclMemAlloc + ncclCommWindowRegister, peers reached
 *                              through their LSA pointers over NVLink / NVSwitch; in-process: the
 *                              graphs' buffers) and kernels do the exchange -- publish the survivor
 *                              count into every peer's window, compute every rank's plan on the
 *                              device (the same plan as dycl_rebalance_plan), store the surplus
 *                              rows straight into the receivers' windows, release / acquire flags
 *                              per level and epoch -- with no host synchronisation; results come
 *                              home the same way.  Same outputs, bitwise.  The window (allocated at
 *                              the first rebalanced exit, collectively) holds max_batch rows of the
 *                              largest exit input plus per-level results; at most 8 ranks and 8
 *                              rebalanced exits; a peer that never arrives is reported (after
 *                              ~20 s) by dycl_rebalance_stats as DYCL_E_NCCL instead of hanging.
 * Errors: INVALID_ARG, STATE (no communicator), UNSUPPORTED (world > 8), OOM. */
enum { DYCL_REBALANCE_MODE_HOST = 0, DYCL_REBALANCE_MODE_DEVICE = 1 };
dycl_status dycl_set_rebalance_mode(dycl_graph g, int mode);
/* Rows this rank sent to / received from other ranks during its last dycl_run. */
dycl_status dycl_rebalance_stats(dycl_graph g, int64_t* rows_sent, int64_t* rows_received);
/* NCCL bootstrap for callers without a communicator: rank 0 gets a 128-byte unique id, shares
 * it out of band, every rank calls dycl_nccl_comm_init_rank (collective). */
dycl_status dycl_nccl_get_unique_id(uint8_t out[128]);
dycl_status dycl_nccl_comm_init_rank(const uint8_t id[128], int rank, int world, int cuda_device, void** comm);
dycl_status dycl_nccl_comm_destroy(void* comm);

/* Survivor rebalancing plan after an exit point: given every rank's
 * survivor count counts[0..world-1], the target is T = ceil(S / world), S = sum(counts).
 * Ranks with more than T survivors send their LAST (count - T) rows, in order, to the
 * ranks with fewer than T, matched in rank order (surplus rank ascending x deficit rank
 * ascending).  Received rows are appended after a rank's own survivors in source-rank
 * order.  For `rank`: send[j] = rows sent to rank j (taken from the tail, destination
 * rank ascending), recv[j] = rows received from rank j, *new_count = rows held after.
 * Pure host function (no device, no communicator); deterministic.  Errors: INVALID_ARG. */
dycl_status dycl_rebalance_plan(const int32_t* counts, int world, int rank, int32_t* send, int32_t* recv,
                                int32_t* new_count);

/* ---------------------------------------------- generative DyNN (config 4) --- */
/* A sequence-to-sequence Transformer decoded greedily under a per-sequence loop guard:
 * the paper's generative DyNNs (AttentionNet), whose `If` node tests the
 * output token to decide whether generation is complete (L265), with the constant
 * maximum-iteration flag the paper prescribes (L267-268).  Rewritten form: an encoder
 * sub-network run once, a decoder-step sub-network + LM head run inside the guarded
 * loop; per step the guard is evaluated on the device and the still-active sequences
 * are compacted (KV caches stay in slot order), so the loop has no host round trip.
 * Post-LN layers (x = LN(x + SA(x)); [x = LN(x + CA(x, mem))]; x = LN(x + FFN(x))),
 * ReLU FFN, sinusoidal PE, embeddings x sqrt(d_model), head dim 64, no final norm. */
typedef struct dycl_s2s_s* dycl_s2s;
typedef struct {
  int vocab, d_model, heads, d_ff, enc_layers, dec_layers;
  int src_len;           /* <= 64, every source sequence has exactly this length   */
  int max_len;           /* <= 64, the loop's constant iteration bound (L267)      */
  int pad, bos, eos;
} dycl_s2s_config;
/* Weights of one layer (host pointers, copied).  bf16 matrices are [n_out][n_in];
 * q|k|v stacked in wqkv [3d][d]; cross-attention: wq2 [d][d], k|v stacked in wkv2 [2d][d].
 * ln_sa / ln_ca / ln_ff: LayerNorm after self-attention / cross-attention (decoder only,
 * NULL for encoder layers) / feed-forward; gamma, beta fp32 [d]; eps 1e-5. */
typedef struct {
  const uint16_t* wqkv; const float* bqkv;
  const uint16_t* wo;   const float* bo;
  const float* ln_sa_g; const float* ln_sa_b;
  const uint16_t* wq2;  const float* bq2;
  const uint16_t* wkv2; const float* bkv2;
  const uint16_t* wo2;  const float* bo2;
  const float* ln_ca_g; const float* ln_ca_b;
  const uint16_t* w1;   const float* b1;
  const uint16_t* w2;   const float* b2;
  const float* ln_ff_g; const float* ln_ff_b;
} dycl_s2s_layer;

dycl_status dycl_s2s_create(int cuda_device, const dycl_s2s_config* cfg, dycl_s2s* out);
dycl_status dycl_s2s_destroy(dycl_s2s s);
const char* dycl_s2s_last_error(dycl_s2s s);
/* src_emb, tgt_emb: bf16 [vocab][d_model]. */
dycl_status dycl_s2s_set_embeddings(dycl_s2s s, const uint16_t* src_emb, const uint16_t* tgt_emb);
dycl_status dycl_s2s_add_encoder_layer(dycl_s2s s, const dycl_s2s_layer* w);
dycl_status dycl_s2s_add_decoder_layer(dycl_s2s s, const dycl_s2s_layer* w);
/* Untied LM head: w bf16 [vocab][d_model], b fp32 [vocab]. */
dycl_status dycl_s2s_set_lm_head(dycl_s2s s, const uint16_t* w, const float* b);
/* The loop guard (the logic node on the output token): at step t the EOS logit gets
 * beta * (t + 1 - len_table[src[0]]) added (len_table fp32 [vocab]; pass beta = 0 for the
 * plain argmax guard); tok = argmax (lowest index on ties); a sequence is done after it
 * emits EOS (EOS counted in its length) or after max_len steps; PAD fills the rest. */
dycl_status dycl_s2s_set_loop_guard(dycl_s2s s, const float* len_table, float beta);
/* Numerics (before finalize).  DYCL_PREC_BF16 (default): bf16 tensor-core operands, bf16
 * q/k/v, K/V caches, attention outputs and FFN hidden, fp32 residual stream / LayerNorm /
 * softmax / logits -- graded against the oracle's mirror mode.  DYCL_PREC_BF16X3_PARITY
 * (SURVEY 8(c) "precision modes"): every bf16 tensor is kept as a split pair hi + lo (hi =
 * bf16(v), lo = bf16(v - hi), ~16 significant bits) and every GEMM runs on the tensor cores over
 * K-concatenated operands [A_hi | A_lo] x [W | W] -- the split-bf16 3-pass product, whose
 * A_hi x W_lo term is identically zero because the weights are exact bf16 -- so products are
 * fp32-accurate; graded against the oracle's exact (fp64) mode, where decisions must be
 * bit-exact outside the 1e-3 band.  Twice the GEMM work and the bf16 bytes.  Errors:
 * INVALID_ARG, STATE. */
dycl_status dycl_s2s_set_precision(dycl_s2s s, int precision);
dycl_status dycl_s2s_finalize(dycl_s2s s, int64_t max_batch);
/* Device buffers: src int32 [batch][src_len]; tokens int32 [batch][max_len] (out);
 * lengths int32 [batch] (out); top1 fp32 [batch][max_len] (out, the chosen token's logit,
 * NaN after done) or NULL; logits0 fp32 [batch][vocab] (out, step-0 logits incl. the
 * guard bias) or NULL.  Stream-ordered, no host synchronisation. */
dycl_status dycl_s2s_run(dycl_s2s s, const int32_t* src, int64_t batch, int32_t* tokens, int32_t* lengths,
                         float* top1, float* logits0, void* stream);
/* Host buffers (src, tokens, lengths): H2D copy, run, D2H copy, synchronise. */
dycl_status dycl_s2s_run_host(dycl_s2s s, const int32_t* src_host, int64_t batch, int32_t* tokens_host,
                              int32_t* lengths_host, void* stream);
/* Number of this library's kernels the last run launched. */
dycl_status dycl_s2s_launches(dycl_s2s s, int32_t* out);
/* Per-launch profiling of the generative graph, same contract as dycl_set_profiling /
 * dycl_profile_read (kinds DYCL_K_GEMM / ATTN / LN / ARGMAX / EMBED / COMPACT / INIT);
 * while enabled, runs are issued launch by launch (no CUDA graph) with events around
 * each launch. */
dycl_status dycl_s2s_set_profiling(dycl_s2s s, int enable);
dycl_status dycl_s2s_profile_read(dycl_s2s s, int32_t max_n, int32_t* kind, float* ms,
                                  double* bytes, double* flops, int32_t* n_out);

/* ------------------------------------ image-captioning En-Decoder --- */
/* The paper's En-Decoder ("Image caption / token wise caption generation"; L323:
 * Show, Attend and Tell).  Encoder = an image graph (any dycl_graph) whose final tensor is
 * exported with dycl_io.features: L = H*W annotation vectors of D = C dims.  This graph is the
 * decoder loop (reading R20): h, c = tanh(init_w[:H] mean(a) + b), tanh(init_w[H:] ...);
 * per step q = att_w h + att_b, alpha = softmax_j(a_j . q / sqrt(D)), z = sum alpha_j a_j, one LSTM
 * cell on [emb[y]; z] with h (gate rows i, f, g, o; lstm_w [4H][E + D + H], lstm_b = b_ih + b_hh),
 * logits = out_w h + out_b, greedy argmax (lowest index on ties); the loop guard of
 * dycl_s2s_set_loop_guard's semantics without the length bias: a caption is done after EOS
 * (counted in its length) or max_len steps, PAD after.  Each step runs on the still-active captions
 * only (compacted on the device); no host synchronisation.  bf16 weights [n_out][n_in], fp32 biases;
 * host pointers copied.  Constraints: D == 64, L <= 64, hidden and emb multiples of 64, vocab of
 * 256, max_len <= 64 (else DYCL_E_UNSUPPORTED). */
typedef struct dycl_cap_s* dycl_cap;
typedef struct {
  int vocab, emb, hidden;
  int feat_len, feat_dim;    /* L, D */
  int max_len, pad, bos, eos;
} dycl_cap_config;
dycl_status dycl_cap_create(int cuda_device, const dycl_cap_config* cfg, dycl_cap* out);
dycl_status dycl_cap_destroy(dycl_cap c);
const char* dycl_cap_last_error(dycl_cap c);
dycl_status dycl_cap_set_weights(dycl_cap c, const uint16_t* init_w, const float* init_b, const uint16_t* att_w,
                                 const float* att_b, const uint16_t* emb, const uint16_t* lstm_w,
                                 const float* lstm_b, const uint16_t* out_w, const float* out_b);
dycl_status dycl_cap_finalize(dycl_cap c, int64_t max_batch);
/* features: device bf16 [batch][L][D]; tokens int32 [batch][max_len] (out); lengths int32 [batch]
 * (out); top1 fp32 [batch][max_len] (out, the chosen token's logit, NaN after done) or NULL.
 * Stream-ordered.  Errors: INVALID_ARG, STATE, SHAPE_MISMATCH (batch > max_batch), CUDA. */
dycl_status dycl_cap_run(dycl_cap c, const uint16_t* features, int64_t batch, int32_t* tokens, int32_t* lengths,
                         float* top1, void* stream);
/* Number of this library's kernels the last dycl_cap_run launched. */
dycl_status dycl_cap_launches(dycl_cap c, int32_t* out);

/* ------------------------------------------------------------ test hook ---- */
/* Run ONE conv2d layer (the a1 tensor-core kernel, same code path dycl_run uses)
 * on caller-owned device buffers and synchronise.  For element-wise kernel tests.
 * bf16 tensors use the library's internal channel-planar layout [n][C/8][H][W][8]
 * (DESIGN.md §4); the residual-stream fp32 tensors dycl_run keeps are NHWC.
 *   x   : device bf16 [n][C/8][H][W][8], C % 8 == 0
 *   w   : host bf16 [c_out][k][k][C];  bias: host fp32 [c_out]
 *   res : device bf16 shortcut (channel-planar) or NULL; res_mode 0 none, 1 identity
 *         [n][c_out/8][Ho][Wo][8], 2 option A from [n][c_out/16][2Ho][2Wo][8]
 *   y   : device bf16 [n][c_out/8][Ho][Wo][8]
 *   path: 0 = the kernel dycl_run would pick, 1 = cp.async-fed kernel, 2 = TMA-fed kernel
 *         (CUDA error "operation not supported" if the shape does not qualify),
 *         4 = NHWC layout: x [n][H][W][C], res [n][Ho][Wo][c_out], y [n][Ho][Wo][c_out], run by
 *         the im2col-TMA GEMM (C % 64 == 0, c_out % 64 == 0; the 8-channel stem by the planar
 *         kernels, which coincide with NHWC at C = 8)
 *         5 = path 4 with the row-tap weight copy supplied: 3x3 / stride 1 / pad 1 layers whose
 *         samples tile 128-row GEMM tiles whole (W | 32, c_out = 64) take the GEMM's row-tap
 *         form (horizontal taps along N, lane-shuffle combine)
 * g supplies the device (any created graph).  Errors: INVALID_ARG, UNSUPPORTED, CUDA. */
dycl_status dycl_debug_conv2d(dycl_graph g, int64_t n, int H, int W, int C, const uint16_t* w, const float* bias,
                              int c_out, int k, int stride, int pad, int relu, const void* res, int res_mode,
                              const void* x, void* y, int path);

/* Development hook: with DYCL_TS set in the environment at graph creation, copies the
 * clock64 phase stamps of the last fused-block launch (CTA 0, first 8 samples, 16 slots
 * each) into out128.  Errors: STATE if DYCL_TS was not set. */
dycl_status dycl_debug_timestamps(dycl_graph g, long long* out128);

#ifdef __cplusplus
}
#endif
#endif /* DYCL_H_ */
