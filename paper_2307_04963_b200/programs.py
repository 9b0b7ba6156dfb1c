"""The three DyNNs in their REWRITTEN form, registered through the C ABI.

This is what DyCL's front end would hand to the runtime: the original program
after loop unrolling + constant propagation (Sec. 5.2, Listing 3 ->
Listing 4) and HCFG partitioning (Sec. 5.3, Alg. 1): a chain
of conditional-free sub-networks (tensor nodes) and logic nodes.  Weights come
from the seeded generator (``workloads``); nothing here computes.

Only this registration, the binding and libdycl.so are on the product path.
"""
from __future__ import annotations

import numpy as np

from . import dycl as D

RELU, NONE = D.DYCL_ACT_RELU, D.DYCL_ACT_NONE


class Model:
    """A finalized graph + its I/O geometry.  ``run`` enqueues one batched inference."""

    def __init__(self, g, in_shape, K, max_batch, name):
        self.g, self.in_shape, self.K, self.max_batch, self.name = g, in_shape, K, max_batch, name

    def run(self, x, logits, path, node_counts=None, stream=None, batch=None, global_offset=0, min_margin=None):
        D.dycl_run(self.g, x, x.shape[0] if batch is None else batch, logits, path, node_counts, stream,
                   global_offset, min_margin)

    def run_host(self, x_host, logits_host, path_host, stream=None, global_offset=0, min_margin=None):
        if global_offset == 0 and min_margin is None:
            D.dycl_run_host(self.g, x_host, x_host.shape[0], logits_host, path_host, stream)
        else:
            D.dycl_run_host_ex(self.g, x_host, x_host.shape[0], global_offset, logits_host, path_host, min_margin,
                               stream)

    def close(self):
        if self.g is not None:
            D.dycl_graph_destroy(self.g)
            self.g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _head(g, W, name, c_in, gap=True):
    sn = D.dycl_subnet_begin(g)
    if gap:
        D.dycl_subnet_gap(g, sn)
    w = np.asarray(W[f"{name}.w"])
    D.dycl_subnet_dense(g, sn, c_in, w.shape[0], w, W[f"{name}.b"], NONE, 1)
    D.dycl_subnet_end(g, sn)
    return sn


def _block(g, sn, W, i, c_in, c_out, stride):
    """He basic block: relu(conv2(relu(conv1(h))) + shortcut(h)); option A when shapes change."""
    D.dycl_subnet_block_begin(g, sn)
    D.dycl_subnet_conv2d(g, sn, c_in, c_out, 3, stride, 1, W[f"b{i}.c1.w"], W[f"b{i}.c1.b"], RELU, 0)
    D.dycl_subnet_conv2d(g, sn, c_out, c_out, 3, 1, 1, W[f"b{i}.c2.w"], W[f"b{i}.c2.b"], RELU, 1)


def _block_io(i, per_stage, widths=(16, 32, 64)):
    s = (i - 1) // per_stage
    if s > 0 and (i - 1) % per_stage == 0:
        return widths[s - 1], widths[s], 2
    return widths[s], widths[s], 1


def _create(device, h, w, c, precision):
    g = D.dycl_graph_create(device, h, w, c)
    D.dycl_graph_set_precision(g, precision)
    return g


FP32_STREAM = D.DYCL_PREC_FP32_STREAM


def build_mlp_ee(W, max_batch, device=0, tau=0.9, precision=FP32_STREAM) -> Model:
    """Config 1: x -> [dense+ReLU -> exit head0] -> [dense+ReLU -> exit head1] -> [dense+ReLU -> final head2]."""
    g = _create(device, 1, 1, 64, precision)
    for k in range(3):
        sn = D.dycl_subnet_begin(g)
        D.dycl_subnet_dense(g, sn, 64, 64, W[f"fc{k}.w"], W[f"fc{k}.b"], RELU, 0)
        D.dycl_subnet_end(g, sn)
        D.dycl_seq(g, sn)
        h = _head(g, W, f"head{k}", 64, gap=False)
        if k < 2:
            D.dycl_exit(g, h, tau)
        else:
            D.dycl_final(g, h)
    D.dycl_finalize(g, max_batch)
    return Model(g, (64,), 10, max_batch, "mlp_ee")


def build_sdn_resnet56(W, max_batch, device=0, tau=None, precision=FP32_STREAM) -> Model:
    """Config 2, rewritten: unrolled 27 blocks split at the IC positions (after 5, 11, 16, 22)."""
    tau = float(W["tau"]) if tau is None else tau
    g = _create(device, 32, 32, 3, precision)
    bounds = [0, 5, 11, 16, 22, 27]
    for k in range(5):
        sn = D.dycl_subnet_begin(g)
        if k == 0:
            D.dycl_subnet_conv2d(g, sn, 3, 16, 3, 1, 1, W["stem.w"], W["stem.b"], RELU, 0)
        for i in range(bounds[k] + 1, bounds[k + 1] + 1):
            _block(g, sn, W, i, *_block_io(i, 9))
        D.dycl_subnet_end(g, sn)
        D.dycl_seq(g, sn)
        c = _block_io(bounds[k + 1], 9)[1]
        if k < 4:
            D.dycl_exit(g, _head(g, W, f"ic{k}", c), tau)
        else:
            D.dycl_final(g, _head(g, W, "final", c))
    D.dycl_finalize(g, max_batch)
    return Model(g, (32, 32, 3), 10, max_batch, "sdn_resnet56")


def build_skipnet_resnet38(W, max_batch, device=0, thr=None, precision=FP32_STREAM) -> Model:
    """Config 3, rewritten (Listing 4 style): stem+block1, then per block i=2..18 a gate node."""
    thr = float(W["thr"]) if thr is None else thr
    g = _create(device, 32, 32, 3, precision)
    sn = D.dycl_subnet_begin(g)
    D.dycl_subnet_conv2d(g, sn, 3, 16, 3, 1, 1, W["stem.w"], W["stem.b"], RELU, 0)
    _block(g, sn, W, 1, 16, 16, 1)
    D.dycl_subnet_end(g, sn)
    D.dycl_seq(g, sn)
    for i in range(2, 19):
        ci, co, stride = _block_io(i, 6)
        gate = _head(g, W, f"gate{i}", ci)
        blk = D.dycl_subnet_begin(g)
        _block(g, blk, W, i, ci, co, stride)
        D.dycl_subnet_end(g, blk)
        D.dycl_gate(g, gate, thr, blk)
    D.dycl_final(g, _head(g, W, "final", 64))
    D.dycl_finalize(g, max_batch)
    return Model(g, (32, 32, 3), 10, max_batch, "skipnet_resnet38")


def build_skipnet_rnn_resnet38(W, max_batch, device=0, thr=None, precision=FP32_STREAM) -> Model:
    """SkipNet with the recurrent gate (Table 3 ID 5 "ResNet38 + RNN"), rewritten:
    stem+block1, then per block i=2..18 a recurrent gate node: proj_i = GAP + dense(C_i -> n_in)
    feeds the graph's one LSTM cell, whose state carries across the gates."""
    thr = float(W["thr"]) if thr is None else thr
    n_in, hid = int(W["rnn.n_in"]), int(W["rnn.hidden"])
    g = _create(device, 32, 32, 3, precision)
    D.dycl_rnn_cell(g, n_in, hid, W["rnn.w_ih"], W["rnn.w_hh"], W["rnn.b_ih"], W["rnn.b_hh"])
    sn = D.dycl_subnet_begin(g)
    D.dycl_subnet_conv2d(g, sn, 3, 16, 3, 1, 1, W["stem.w"], W["stem.b"], RELU, 0)
    _block(g, sn, W, 1, 16, 16, 1)
    D.dycl_subnet_end(g, sn)
    D.dycl_seq(g, sn)
    for i in range(2, 19):
        ci, co, stride = _block_io(i, 6)
        proj = _head(g, W, f"proj{i}", ci)
        blk = D.dycl_subnet_begin(g)
        _block(g, blk, W, i, ci, co, stride)
        D.dycl_subnet_end(g, blk)
        D.dycl_gate_rnn(g, proj, W[f"out{i}.w"], float(np.asarray(W[f"out{i}.b"]).reshape(-1)[0]), thr, blk)
    D.dycl_final(g, _head(g, W, "final", 64))
    D.dycl_finalize(g, max_batch)
    return Model(g, (32, 32, 3), 10, max_batch, "skipnet_rnn_resnet38")


R50_LAYERS = (3, 4, 6, 3)
R50_WIDTHS = (64, 128, 256, 512)


def build_resnet50_ee(W, max_batch, device=0, tau=None, precision=FP32_STREAM, hw=224) -> Model:
    """Config 5, rewritten: one sub-network per stage (stem + maxpool fused into the first),
    exits after stages 1-3, final head after stage 4 (1000 classes)."""
    tau = float(W["tau"]) if tau is None else tau
    g = _create(device, hw, hw, 3, precision)
    c_in = 64
    for s in range(1, 5):
        sn = D.dycl_subnet_begin(g)
        if s == 1:
            D.dycl_subnet_conv2d(g, sn, 3, 64, 7, 2, 3, W["stem.w"], W["stem.b"], RELU, 0)
            D.dycl_subnet_maxpool(g, sn, 3, 2, 1)
        w = R50_WIDTHS[s - 1]
        for b in range(R50_LAYERS[s - 1]):
            p = f"s{s}b{b}"
            stride = 2 if (b == 0 and s > 1) else 1
            D.dycl_subnet_block_begin(g, sn)
            D.dycl_subnet_conv2d(g, sn, c_in, w, 1, 1, 0, W[f"{p}.c1.w"], W[f"{p}.c1.b"], RELU, 0)
            D.dycl_subnet_conv2d(g, sn, w, w, 3, stride, 1, W[f"{p}.c2.w"], W[f"{p}.c2.b"], RELU, 0)
            if b == 0:
                D.dycl_subnet_projection(g, sn, c_in, 4 * w, stride, W[f"{p}.proj.w"], W[f"{p}.proj.b"])
            D.dycl_subnet_conv2d(g, sn, w, 4 * w, 1, 1, 0, W[f"{p}.c3.w"], W[f"{p}.c3.b"], RELU, 1)
            c_in = 4 * w
        D.dycl_subnet_end(g, sn)
        D.dycl_seq(g, sn)
        if s < 4:
            D.dycl_exit(g, _head(g, W, f"ic{s - 1}", c_in), tau)
        else:
            D.dycl_final(g, _head(g, W, "final", c_in))
    D.dycl_finalize(g, max_batch)
    return Model(g, (hw, hw, 3), 1000, max_batch, "resnet50_ee")


class Seq2Seq:
    """Config 4: the generative graph (encoder once, decoder step + LM head under the loop guard)."""

    def __init__(self, h, cfg, max_batch):
        self.h, self.cfg, self.max_batch = h, cfg, max_batch

    def run(self, src, tokens, lengths, top1=None, logits0=None, stream=None, batch=None):
        D.dycl_s2s_run(self.h, src, src.shape[0] if batch is None else batch, tokens, lengths, top1, logits0, stream)

    def run_host(self, src_host, tokens_host, lengths_host, stream=None):
        D.dycl_s2s_run_host(self.h, src_host, src_host.shape[0], tokens_host, lengths_host, stream)

    def close(self):
        if self.h is not None:
            D.dycl_s2s_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_seq2seq(W, cfg, max_batch, device=0, precision=D.DYCL_PREC_BF16) -> Seq2Seq:
    """Config 4, rewritten: encoder sub-network + decoder-step sub-network + LM head, with the
    EOS / length guard registered as the loop's logic node.  precision: DYCL_PREC_BF16
    (production) or DYCL_PREC_BF16X3_PARITY (fp32-accurate split-bf16 products)."""
    cfg = dict(cfg)
    cfg.setdefault("d_model", cfg.get("d"))
    h = D.dycl_s2s_create(device, cfg)
    if precision != D.DYCL_PREC_BF16:
        D.dycl_s2s_set_precision(h, precision)
    D.dycl_s2s_set_embeddings(h, W["src_emb"], W["tgt_emb"])
    for l in range(cfg["enc_layers"]):
        p = f"enc{l}."
        D.dycl_s2s_add_encoder_layer(h, dict(
            wqkv=W[p + "wqkv"], bqkv=W[p + "bqkv"], wo=W[p + "wo"], bo=W[p + "bo"],
            ln_sa_g=W[p + "ln1.g"], ln_sa_b=W[p + "ln1.b"], w1=W[p + "w1"], b1=W[p + "b1"],
            w2=W[p + "w2"], b2=W[p + "b2"], ln_ff_g=W[p + "ln2.g"], ln_ff_b=W[p + "ln2.b"]))
    for l in range(cfg["dec_layers"]):
        p = f"dec{l}."
        D.dycl_s2s_add_decoder_layer(h, dict(
            wqkv=W[p + "wqkv"], bqkv=W[p + "bqkv"], wo=W[p + "wo"], bo=W[p + "bo"],
            ln_sa_g=W[p + "ln1.g"], ln_sa_b=W[p + "ln1.b"], wq2=W[p + "wq2"], bq2=W[p + "bq2"],
            wkv2=W[p + "wkv2"], bkv2=W[p + "bkv2"], wo2=W[p + "wo2"], bo2=W[p + "bo2"],
            ln_ca_g=W[p + "ln2.g"], ln_ca_b=W[p + "ln2.b"], w1=W[p + "w1"], b1=W[p + "b1"],
            w2=W[p + "w2"], b2=W[p + "b2"], ln_ff_g=W[p + "ln3.g"], ln_ff_b=W[p + "ln3.b"]))
    D.dycl_s2s_set_lm_head(h, W["lm.w"], W["lm.b"])
    D.dycl_s2s_set_loop_guard(h, W["len_table"], float(W["beta"]))
    D.dycl_s2s_finalize(h, max_batch)
    return Seq2Seq(h, cfg, max_batch)


class Caption:
    """The captioning En-Decoder (reading R20): the encoder image graph (its final
    tensor exported through dycl_io.features) chained with the decoder loop graph (dycl_cap_*) --
    the host program P_Host of Listing 2: run the encoder sub-network, then the guarded loop."""

    def __init__(self, enc, h, cfg, max_batch):
        self.enc, self.h, self.cfg, self.max_batch = enc, h, cfg, max_batch

    def run(self, x, tokens, lengths, top1=None, stream=None, features=None):
        """x: CUDA fp32 [B][32][32][3]; tokens int32 [B][max_len], lengths int32 [B], top1 fp32
        [B][max_len] or None (outputs).  Returns the encoder's annotation vectors (bf16 bits)."""
        import torch
        B = x.shape[0]
        feats = features if features is not None else \
            torch.empty((B, self.cfg["L"], self.cfg["D"]), dtype=torch.int16, device=x.device)
        lg = torch.empty((B, self.enc.K), device=x.device)
        pa = torch.empty(B, dtype=torch.int32, device=x.device)
        D.dycl_run(self.enc.g, x, B, lg, pa, stream=stream, features=feats)
        D.dycl_cap_run(self.h, feats, B, tokens, lengths, top1, stream)
        return feats

    def close(self):
        if self.h is not None:
            D.dycl_cap_destroy(self.h)
            self.h = None
        self.enc.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_caption(W, cfg, max_batch, device=0, precision=FP32_STREAM) -> Caption:
    """Captioning En-Decoder, rewritten: the encoder sub-network (the CIFAR ResNet-38 trunk, one
    conditional-free subnet; a small head closes the image graph, its output unused) and the
    decoder-step sub-networks + LM head under the loop guard (dycl_cap_*)."""
    g = _create(device, 32, 32, 3, precision)
    sn = D.dycl_subnet_begin(g)
    D.dycl_subnet_conv2d(g, sn, 3, 16, 3, 1, 1, W["stem.w"], W["stem.b"], RELU, 0)
    for i in range(1, 19):
        _block(g, sn, W, i, *_block_io(i, 6))
    D.dycl_subnet_end(g, sn)
    D.dycl_seq(g, sn)
    head = D.dycl_subnet_begin(g)
    D.dycl_subnet_gap(g, head)
    D.dycl_subnet_dense(g, head, 64, 16, np.zeros((16, 64), np.uint16), np.zeros(16, np.float32), NONE, 1)
    D.dycl_subnet_end(g, head)
    D.dycl_final(g, head)
    D.dycl_finalize(g, max_batch)
    enc = Model(g, (32, 32, 3), 16, max_batch, "caption_encoder")
    h = D.dycl_cap_create(device, cfg)
    D.dycl_cap_set_weights(h, W["init.w"], W["init.b"], W["att.w"], W["att.b"], W["emb"], W["lstm.w"], W["lstm.b"],
                           W["out.w"], W["out.b"])
    D.dycl_cap_finalize(h, max_batch)
    return Caption(enc, h, dict(cfg), max_batch)


BUILDERS = {1: build_mlp_ee, 2: build_sdn_resnet56, 3: build_skipnet_resnet38, 5: build_resnet50_ee}
