"""Thin ctypes binding of libdycl.so (include/dycl.h): same names, argument marshalling only.

Every step of the path runs in libdycl's kernels.  There is no CPU fallback:
if the shared library is missing, or no sm_100 device is present, calls raise.
Device buffers are passed as torch tensors (data_ptr) -- PyTorch is used only
for device memory and streams.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdycl.so")

DYCL_ACT_NONE = 0
DYCL_ACT_RELU = 1
KIND_NAMES = {0: "input", 1: "conv", 2: "head", 3: "compact", 4: "gather", 5: "scatter", 6: "init", 7: "pool",
              8: "block", 9: "gemm", 10: "attn", 11: "ln", 12: "argmax", 13: "embed"}

_STATUS = {0: "DYCL_OK", -1: "DYCL_E_INVALID_ARG", -2: "DYCL_E_SHAPE_MISMATCH", -3: "DYCL_E_SIGNATURE",
           -4: "DYCL_E_SHAPE_JOIN", -5: "DYCL_E_STATE", -6: "DYCL_E_UNSUPPORTED", -7: "DYCL_E_OOM",
           -8: "DYCL_E_CUDA", -9: "DYCL_E_NCCL"}


class DyclError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class dycl_io(ctypes.Structure):
    _fields_ = [("input", ctypes.c_void_p), ("batch", ctypes.c_int64), ("logits", ctypes.c_void_p),
                ("path", ctypes.c_void_p), ("node_counts", ctypes.c_void_p), ("global_offset", ctypes.c_int64),
                ("min_margin", ctypes.c_void_p), ("features", ctypes.c_void_p)]


DYCL_REBALANCE_NONE = 0
DYCL_REBALANCE_ALL = -1
DYCL_REBALANCE_MODE_HOST = 0
DYCL_REBALANCE_MODE_DEVICE = 1


class dycl_cap_config(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in ("vocab", "emb", "hidden", "feat_len", "feat_dim", "max_len", "pad", "bos",
                                            "eos")]


class dycl_s2s_config(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in ("vocab", "d_model", "heads", "d_ff", "enc_layers", "dec_layers",
                                            "src_len", "max_len", "pad", "bos", "eos")]


class dycl_s2s_layer(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in (
        "wqkv", "bqkv", "wo", "bo", "ln_sa_g", "ln_sa_b", "wq2", "bq2", "wkv2", "bkv2", "wo2", "bo2",
        "ln_ca_g", "ln_ca_b", "w1", "b1", "w2", "b2", "ln_ff_g", "ln_ff_b")]


_lib = None
EXPORTS = [
    "dycl_s2s_create", "dycl_s2s_destroy", "dycl_s2s_last_error", "dycl_s2s_set_embeddings",
    "dycl_s2s_add_encoder_layer", "dycl_s2s_add_decoder_layer", "dycl_s2s_set_lm_head", "dycl_s2s_set_loop_guard",
    "dycl_s2s_finalize", "dycl_s2s_run", "dycl_s2s_run_host", "dycl_s2s_launches",
    "dycl_s2s_set_profiling", "dycl_s2s_profile_read",
    "dycl_graph_create", "dycl_graph_set_precision", "dycl_graph_destroy", "dycl_last_error", "dycl_subnet_begin", "dycl_subnet_block_begin",
    "dycl_subnet_conv2d", "dycl_subnet_dense", "dycl_subnet_gap", "dycl_subnet_projection", "dycl_subnet_maxpool", "dycl_subnet_end", "dycl_seq", "dycl_exit",
    "dycl_gate", "dycl_rnn_cell", "dycl_gate_rnn", "dycl_final", "dycl_finalize", "dycl_run", "dycl_run_host", "dycl_num_count_slots",
    "dycl_launches_per_run", "dycl_num_classes", "dycl_set_profiling", "dycl_profile_read",
    "dycl_debug_conv2d", "dycl_rebalance_plan", "dycl_debug_timestamps",
    "dycl_run_host_ex", "dycl_set_comm", "dycl_local_group_create", "dycl_local_group_destroy",
    "dycl_set_comm_local", "dycl_set_rebalance_mode", "dycl_rebalance_stats", "dycl_nccl_get_unique_id", "dycl_nccl_comm_init_rank",
    "dycl_nccl_comm_destroy", "dycl_s2s_set_precision",
    "dycl_cap_create", "dycl_cap_destroy", "dycl_cap_last_error", "dycl_cap_set_weights", "dycl_cap_finalize",
    "dycl_cap_run", "dycl_cap_launches",
]


def lib():
    """Load libdycl.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, f32 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_float
        P16 = ctypes.POINTER(ctypes.c_uint16)
        Pf = ctypes.POINTER(ctypes.c_float)
        Pi = ctypes.POINTER(ctypes.c_int32)
        Pd = ctypes.POINTER(ctypes.c_double)
        sig = {
            "dycl_graph_create": [i32, i32, i32, i32, ctypes.POINTER(vp)],
            "dycl_graph_destroy": [vp],
            "dycl_graph_set_precision": [vp, i32],
            "dycl_subnet_begin": [vp, Pi],
            "dycl_subnet_block_begin": [vp, i32],
            "dycl_subnet_conv2d": [vp, i32, i32, i32, i32, i32, i32, P16, Pf, i32, i32],
            "dycl_subnet_dense": [vp, i32, i32, i32, P16, Pf, i32, i32],
            "dycl_subnet_gap": [vp, i32],
            "dycl_subnet_projection": [vp, i32, i32, i32, i32, P16, Pf],
            "dycl_subnet_maxpool": [vp, i32, i32, i32, i32],
            "dycl_subnet_end": [vp, i32],
            "dycl_seq": [vp, i32],
            "dycl_exit": [vp, i32, f32],
            "dycl_gate": [vp, i32, f32, i32],
            "dycl_rnn_cell": [vp, i32, i32, Pf, Pf, Pf, Pf],
            "dycl_gate_rnn": [vp, i32, Pf, f32, f32, i32],
            "dycl_final": [vp, i32],
            "dycl_finalize": [vp, i64],
            "dycl_run": [vp, ctypes.POINTER(dycl_io), vp],
            "dycl_run_host": [vp, vp, i64, vp, vp, vp],
            "dycl_num_count_slots": [vp, Pi],
            "dycl_launches_per_run": [vp, Pi],
            "dycl_num_classes": [vp, Pi],
            "dycl_set_profiling": [vp, i32],
            "dycl_profile_read": [vp, i32, Pi, Pf, Pd, Pd, Pi],
            "dycl_rebalance_plan": [Pi, i32, i32, Pi, Pi, Pi],
            "dycl_debug_timestamps": [vp, ctypes.POINTER(ctypes.c_longlong)],
            "dycl_debug_conv2d": [vp, i64, i32, i32, i32, P16, Pf, i32, i32, i32, i32, i32, vp, i32, vp, vp, i32],
            "dycl_run_host_ex": [vp, vp, i64, i64, vp, vp, vp, vp],
            "dycl_set_comm": [vp, vp, i32, i32, i32],
            "dycl_local_group_create": [i32, ctypes.POINTER(vp)],
            "dycl_local_group_destroy": [vp],
            "dycl_set_comm_local": [vp, vp, i32, i32],
            "dycl_set_rebalance_mode": [vp, i32],
            "dycl_rebalance_stats": [vp, ctypes.POINTER(i64), ctypes.POINTER(i64)],
            "dycl_nccl_get_unique_id": [ctypes.POINTER(ctypes.c_uint8)],
            "dycl_nccl_comm_init_rank": [ctypes.POINTER(ctypes.c_uint8), i32, i32, i32, ctypes.POINTER(vp)],
            "dycl_nccl_comm_destroy": [vp],
        }
        sig.update({
            "dycl_s2s_create": [i32, ctypes.POINTER(dycl_s2s_config), ctypes.POINTER(vp)],
            "dycl_s2s_destroy": [vp],
            "dycl_s2s_set_embeddings": [vp, vp, vp],
            "dycl_s2s_add_encoder_layer": [vp, ctypes.POINTER(dycl_s2s_layer)],
            "dycl_s2s_add_decoder_layer": [vp, ctypes.POINTER(dycl_s2s_layer)],
            "dycl_s2s_set_lm_head": [vp, vp, vp],
            "dycl_s2s_set_loop_guard": [vp, vp, f32],
            "dycl_s2s_finalize": [vp, i64],
            "dycl_s2s_set_precision": [vp, i32],
            "dycl_s2s_run": [vp, vp, i64, vp, vp, vp, vp, vp],
            "dycl_s2s_run_host": [vp, vp, i64, vp, vp, vp],
            "dycl_s2s_launches": [vp, Pi],
            "dycl_s2s_set_profiling": [vp, i32],
            "dycl_s2s_profile_read": [vp, i32, Pi, Pf, Pd, Pd, Pi],
        })
        sig.update({
            "dycl_cap_create": [i32, ctypes.POINTER(dycl_cap_config), ctypes.POINTER(vp)],
            "dycl_cap_destroy": [vp],
            "dycl_cap_set_weights": [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp],
            "dycl_cap_finalize": [vp, i64],
            "dycl_cap_run": [vp, vp, i64, vp, vp, vp, vp],
            "dycl_cap_launches": [vp, Pi],
        })
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        L.dycl_last_error.argtypes = [vp]
        L.dycl_last_error.restype = ctypes.c_char_p
        L.dycl_cap_last_error.argtypes = [vp]
        L.dycl_cap_last_error.restype = ctypes.c_char_p
        L.dycl_s2s_last_error.argtypes = [vp]
        L.dycl_s2s_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _ck(status, g=None):
    if status != 0:
        msg = lib().dycl_last_error(g).decode(errors="replace")
        raise DyclError(status, msg)


def _u16(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.uint16))
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint16))


def _f32(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def _stream_ptr(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(int(getattr(stream, "cuda_stream", stream)))


# ---------------------------------------------------------------- C-ABI names
def dycl_graph_create(cuda_device: int, in_h: int, in_w: int, in_c: int):
    h = ctypes.c_void_p()
    _ck(lib().dycl_graph_create(cuda_device, in_h, in_w, in_c, ctypes.byref(h)), None)
    return h


DYCL_PREC_BF16 = 0
DYCL_PREC_FP32_STREAM = 1
DYCL_PREC_BF16X3_PARITY = 2


def dycl_graph_set_precision(g, precision):
    _ck(lib().dycl_graph_set_precision(g, int(precision)), g)


def dycl_graph_destroy(g):
    _ck(lib().dycl_graph_destroy(g), None)


def dycl_last_error(g=None) -> str:
    return lib().dycl_last_error(g).decode(errors="replace")


def dycl_subnet_begin(g) -> int:
    n = ctypes.c_int32()
    _ck(lib().dycl_subnet_begin(g, ctypes.byref(n)), g)
    return n.value


def dycl_subnet_block_begin(g, sn):
    _ck(lib().dycl_subnet_block_begin(g, sn), g)


def dycl_subnet_conv2d(g, sn, c_in, c_out, k, stride, pad, w_bf16, bias, act, residual):
    w, wp = _u16(w_bf16)
    b, bp = _f32(bias)
    _ck(lib().dycl_subnet_conv2d(g, sn, c_in, c_out, k, stride, pad, wp, bp, act, int(residual)), g)


def dycl_subnet_dense(g, sn, n_in, n_out, w_bf16, bias, act, out_fp32):
    w, wp = _u16(w_bf16)
    b, bp = _f32(bias)
    _ck(lib().dycl_subnet_dense(g, sn, n_in, n_out, wp, bp, act, int(out_fp32)), g)


def dycl_subnet_projection(g, sn, c_in, c_out, stride, w_bf16, bias):
    w, wp = _u16(w_bf16)
    b, bp = _f32(bias)
    _ck(lib().dycl_subnet_projection(g, sn, c_in, c_out, stride, wp, bp), g)


def dycl_subnet_maxpool(g, sn, k, stride, pad):
    _ck(lib().dycl_subnet_maxpool(g, sn, k, stride, pad), g)


def dycl_subnet_gap(g, sn):
    _ck(lib().dycl_subnet_gap(g, sn), g)


def dycl_subnet_end(g, sn):
    _ck(lib().dycl_subnet_end(g, sn), g)


def dycl_seq(g, sn):
    _ck(lib().dycl_seq(g, sn), g)


def dycl_exit(g, head_sn, tau):
    _ck(lib().dycl_exit(g, head_sn, float(tau)), g)


def dycl_gate(g, gate_sn, thr, then_sn):
    _ck(lib().dycl_gate(g, gate_sn, float(thr), then_sn), g)


def dycl_rnn_cell(g, n_in, hidden, w_ih, w_hh, b_ih, b_hh):
    a, pa = _f32(w_ih)
    b, pb = _f32(w_hh)
    c, pc = _f32(b_ih)
    d, pd = _f32(b_hh)
    _ck(lib().dycl_rnn_cell(g, n_in, hidden, pa, pb, pc, pd), g)


def dycl_gate_rnn(g, proj_sn, w_out, b_out, thr, then_sn):
    a, pa = _f32(w_out)
    _ck(lib().dycl_gate_rnn(g, proj_sn, pa, float(b_out), float(thr), then_sn), g)


def dycl_final(g, head_sn):
    _ck(lib().dycl_final(g, head_sn), g)


def dycl_finalize(g, max_batch):
    _ck(lib().dycl_finalize(g, int(max_batch)), g)


def dycl_run(g, input, batch, logits, path, node_counts=None, stream=None, global_offset=0, min_margin=None,
             features=None):
    """input/logits/path/node_counts/min_margin/features: CUDA torch tensors (fp32, fp32, int32, int32,
    fp32, bf16 bits as int16)."""
    io = dycl_io(input.data_ptr(), int(batch), logits.data_ptr(), path.data_ptr(),
                 node_counts.data_ptr() if node_counts is not None else None, int(global_offset),
                 min_margin.data_ptr() if min_margin is not None else None,
                 features.data_ptr() if features is not None else None)
    _ck(lib().dycl_run(g, ctypes.byref(io), _stream_ptr(stream)), g)


def dycl_run_host(g, input_host, batch, logits_host, path_host, stream=None):
    """Host buffers (torch CPU tensors, pinned or not, or numpy arrays)."""
    def ptr(t):
        return t.data_ptr() if hasattr(t, "data_ptr") else t.ctypes.data
    _ck(lib().dycl_run_host(g, ctypes.c_void_p(ptr(input_host)), int(batch), ctypes.c_void_p(ptr(logits_host)),
                            ctypes.c_void_p(ptr(path_host)), _stream_ptr(stream)), g)


def dycl_run_host_ex(g, input_host, batch, global_offset, logits_host, path_host, min_margin_host=None,
                     stream=None):
    def ptr(t):
        return t.data_ptr() if hasattr(t, "data_ptr") else t.ctypes.data
    _ck(lib().dycl_run_host_ex(g, ctypes.c_void_p(ptr(input_host)), int(batch), int(global_offset),
                               ctypes.c_void_p(ptr(logits_host)), ctypes.c_void_p(ptr(path_host)),
                               ctypes.c_void_p(ptr(min_margin_host)) if min_margin_host is not None else None,
                               _stream_ptr(stream)), g)


def dycl_set_comm(g, nccl_comm_ptr, rank, world, rebalance_policy=DYCL_REBALANCE_ALL):
    """nccl_comm_ptr: an ncclComm_t as an int (e.g. ProcessGroupNCCL._comm_ptr())."""
    _ck(lib().dycl_set_comm(g, ctypes.c_void_p(int(nccl_comm_ptr) if nccl_comm_ptr else 0), int(rank), int(world),
                            int(rebalance_policy)), g)


def dycl_local_group_create(world):
    h = ctypes.c_void_p()
    _ck(lib().dycl_local_group_create(int(world), ctypes.byref(h)), None)
    return h


def dycl_local_group_destroy(grp):
    _ck(lib().dycl_local_group_destroy(grp), None)


def dycl_set_comm_local(g, grp, rank, rebalance_policy=DYCL_REBALANCE_ALL):
    _ck(lib().dycl_set_comm_local(g, grp, int(rank), int(rebalance_policy)), g)


def dycl_set_rebalance_mode(g, mode):
    _ck(lib().dycl_set_rebalance_mode(g, int(mode)), g)


def dycl_rebalance_stats(g):
    a, b = ctypes.c_int64(), ctypes.c_int64()
    _ck(lib().dycl_rebalance_stats(g, ctypes.byref(a), ctypes.byref(b)), g)
    return a.value, b.value


def dycl_nccl_get_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _ck(lib().dycl_nccl_get_unique_id(buf), None)
    return bytes(buf)


def dycl_nccl_comm_init_rank(uid: bytes, rank, world, cuda_device):
    buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
    h = ctypes.c_void_p()
    _ck(lib().dycl_nccl_comm_init_rank(buf, int(rank), int(world), int(cuda_device), ctypes.byref(h)), None)
    return h


def dycl_nccl_comm_destroy(comm):
    _ck(lib().dycl_nccl_comm_destroy(comm), None)


def dycl_num_count_slots(g) -> int:
    n = ctypes.c_int32()
    _ck(lib().dycl_num_count_slots(g, ctypes.byref(n)), g)
    return n.value


def dycl_launches_per_run(g) -> int:
    n = ctypes.c_int32()
    _ck(lib().dycl_launches_per_run(g, ctypes.byref(n)), g)
    return n.value


def dycl_num_classes(g) -> int:
    n = ctypes.c_int32()
    _ck(lib().dycl_num_classes(g, ctypes.byref(n)), g)
    return n.value


def dycl_set_profiling(g, enable):
    _ck(lib().dycl_set_profiling(g, int(bool(enable))), g)


def dycl_profile_read(g, max_n=4096):
    kind = (ctypes.c_int32 * max_n)()
    ms = (ctypes.c_float * max_n)()
    by = (ctypes.c_double * max_n)()
    fl = (ctypes.c_double * max_n)()
    n = ctypes.c_int32()
    _ck(lib().dycl_profile_read(g, max_n, kind, ms, by, fl, ctypes.byref(n)), g)
    m = min(n.value, max_n)
    return [dict(kind=KIND_NAMES[kind[i]], ms=ms[i], bytes=by[i], flops=fl[i]) for i in range(m)]


def dycl_debug_conv2d(g, x, n, H, W, C, w_bf16, bias, c_out, k, stride, pad, relu, res, res_mode, y, path=0):
    w, wp = _u16(w_bf16)
    b, bp = _f32(bias)
    _ck(lib().dycl_debug_conv2d(g, int(n), H, W, C, wp, bp, c_out, k, stride, pad, int(relu),
                                ctypes.c_void_p(res.data_ptr() if res is not None else 0), int(res_mode),
                                ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()), int(path)), g)


# ------------------------------------------------------------ generative graph (config 4)
def _s2s_ck(status, s=None):
    if status != 0:
        raise DyclError(status, lib().dycl_s2s_last_error(s).decode(errors="replace"))


def _hp(a, dtype):
    """Host pointer of a contiguous numpy copy (the caller keeps the returned array alive)."""
    a = np.ascontiguousarray(np.asarray(a, dtype=dtype))
    return a, ctypes.c_void_p(a.ctypes.data)


def dycl_s2s_create(cuda_device, cfg: dict):
    c = dycl_s2s_config(**{f: int(cfg[f]) for f, _ in dycl_s2s_config._fields_})
    h = ctypes.c_void_p()
    _s2s_ck(lib().dycl_s2s_create(cuda_device, ctypes.byref(c), ctypes.byref(h)))
    return h


def dycl_s2s_destroy(s):
    _s2s_ck(lib().dycl_s2s_destroy(s))


def dycl_s2s_last_error(s=None) -> str:
    return lib().dycl_s2s_last_error(s).decode(errors="replace")


def dycl_s2s_set_embeddings(s, src_emb, tgt_emb):
    a, pa = _hp(src_emb, np.uint16)
    b, pb = _hp(tgt_emb, np.uint16)
    _s2s_ck(lib().dycl_s2s_set_embeddings(s, pa, pb), s)


def _layer_struct(w: dict):
    keep = []
    kw = {}
    for f, _ in dycl_s2s_layer._fields_:
        v = w.get(f)
        if v is None:
            kw[f] = None
            continue
        a, p = _hp(v, np.uint16 if np.asarray(v).dtype == np.uint16 else np.float32)
        keep.append(a)
        kw[f] = p.value
    return dycl_s2s_layer(**kw), keep


def dycl_s2s_add_encoder_layer(s, w: dict):
    st, keep = _layer_struct(w)
    _s2s_ck(lib().dycl_s2s_add_encoder_layer(s, ctypes.byref(st)), s)


def dycl_s2s_add_decoder_layer(s, w: dict):
    st, keep = _layer_struct(w)
    _s2s_ck(lib().dycl_s2s_add_decoder_layer(s, ctypes.byref(st)), s)


def dycl_s2s_set_lm_head(s, w, b):
    a, pa = _hp(w, np.uint16)
    c, pc = _hp(b, np.float32)
    _s2s_ck(lib().dycl_s2s_set_lm_head(s, pa, pc), s)


def dycl_s2s_set_loop_guard(s, len_table, beta):
    if len_table is None:
        _s2s_ck(lib().dycl_s2s_set_loop_guard(s, None, float(beta)), s)
        return
    a, pa = _hp(len_table, np.float32)
    _s2s_ck(lib().dycl_s2s_set_loop_guard(s, pa, float(beta)), s)


def dycl_s2s_set_precision(s, precision):
    _s2s_ck(lib().dycl_s2s_set_precision(s, int(precision)), s)


def dycl_s2s_finalize(s, max_batch):
    _s2s_ck(lib().dycl_s2s_finalize(s, int(max_batch)), s)


def dycl_s2s_run(s, src, batch, tokens, lengths, top1=None, logits0=None, stream=None):
    """Device tensors: src int32 [B][S], tokens int32 [B][L], lengths int32 [B], top1 fp32 [B][L], logits0 [B][V]."""
    ptr = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
    _s2s_ck(lib().dycl_s2s_run(s, ptr(src), int(batch), ptr(tokens), ptr(lengths), ptr(top1), ptr(logits0),
                               _stream_ptr(stream)), s)


def dycl_s2s_run_host(s, src_host, batch, tokens_host, lengths_host, stream=None):
    def p(t):
        return ctypes.c_void_p(t.data_ptr() if hasattr(t, "data_ptr") else t.ctypes.data)
    _s2s_ck(lib().dycl_s2s_run_host(s, p(src_host), int(batch), p(tokens_host), p(lengths_host),
                                    _stream_ptr(stream)), s)


def dycl_s2s_set_profiling(s, enable):
    _s2s_ck(lib().dycl_s2s_set_profiling(s, int(bool(enable))), s)


def dycl_s2s_profile_read(s, max_n=8192):
    kind = (ctypes.c_int32 * max_n)()
    ms = (ctypes.c_float * max_n)()
    by = (ctypes.c_double * max_n)()
    fl = (ctypes.c_double * max_n)()
    n = ctypes.c_int32()
    _s2s_ck(lib().dycl_s2s_profile_read(s, max_n, kind, ms, by, fl, ctypes.byref(n)), s)
    m = min(n.value, max_n)
    return [dict(kind=KIND_NAMES[kind[i]], ms=ms[i], bytes=by[i], flops=fl[i]) for i in range(m)]


def dycl_s2s_launches(s) -> int:
    n = ctypes.c_int32()
    _s2s_ck(lib().dycl_s2s_launches(s, ctypes.byref(n)), s)
    return n.value


def dycl_rebalance_plan(counts, rank):
    """-> (send [world], recv [world], new_count) for `rank` (host function, no device)."""
    c = np.ascontiguousarray(np.asarray(counts, dtype=np.int32))
    w = len(c)
    snd = np.zeros(w, np.int32)
    rcv = np.zeros(w, np.int32)
    nc = ctypes.c_int32()
    P = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))  # noqa: E731
    _ck(lib().dycl_rebalance_plan(P(c), w, int(rank), P(snd), P(rcv), ctypes.byref(nc)), None)
    return snd, rcv, nc.value


def dycl_debug_timestamps(g):
    buf = (ctypes.c_longlong * 128)()
    _ck(lib().dycl_debug_timestamps(g, buf), g)
    return np.array(buf[:], dtype=np.int64).reshape(8, 16)


# ------------------------------------------------------------------ captioning En-Decoder
def _cap_ck(status, c=None):
    if status != 0:
        raise DyclError(status, lib().dycl_cap_last_error(c).decode(errors="replace"))


def dycl_cap_create(cuda_device, cfg: dict):
    c = dycl_cap_config(*(int(cfg[k]) for k in ("vocab", "emb", "hidden", "L", "D", "max_len", "pad", "bos", "eos")))
    h = ctypes.c_void_p()
    _cap_ck(lib().dycl_cap_create(cuda_device, ctypes.byref(c), ctypes.byref(h)))
    return h


def dycl_cap_destroy(c):
    _cap_ck(lib().dycl_cap_destroy(c), c)


def dycl_cap_last_error(c=None) -> str:
    return lib().dycl_cap_last_error(c).decode(errors="replace")


def dycl_cap_set_weights(c, init_w, init_b, att_w, att_b, emb, lstm_w, lstm_b, out_w, out_b):
    keep = [_hp(init_w, np.uint16), _hp(init_b, np.float32), _hp(att_w, np.uint16), _hp(att_b, np.float32),
            _hp(emb, np.uint16), _hp(lstm_w, np.uint16), _hp(lstm_b, np.float32), _hp(out_w, np.uint16),
            _hp(out_b, np.float32)]
    _cap_ck(lib().dycl_cap_set_weights(c, *[p for _, p in keep]), c)


def dycl_cap_finalize(c, max_batch):
    _cap_ck(lib().dycl_cap_finalize(c, int(max_batch)), c)


def dycl_cap_run(c, features, batch, tokens, lengths, top1=None, stream=None):
    _cap_ck(lib().dycl_cap_run(c, ctypes.c_void_p(features.data_ptr()), int(batch), ctypes.c_void_p(tokens.data_ptr()),
                               ctypes.c_void_p(lengths.data_ptr()),
                               ctypes.c_void_p(top1.data_ptr()) if top1 is not None else None, _stream_ptr(stream)), c)


def dycl_cap_launches(c) -> int:
    n = ctypes.c_int32()
    _cap_ck(lib().dycl_cap_launches(c, ctypes.byref(n)), c)
    return n.value
