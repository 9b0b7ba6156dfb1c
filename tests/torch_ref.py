"""Independent library compositions used to PIN the oracle (tests only).

Static networks written with torch CPU fp64 ops (NCHW, F.conv2d, F.pad), the
special cases the dynamic programs reduce to when their predicates are forced:
tau > 1 (never exit) -> the static ResNet; tau <= 1/K -> the prefix up to IC1;
gate bias +inf -> plain ResNet-38; -inf -> stem + block 1 + shortcuts.
Nothing here imports oracle/ code.
"""
import numpy as np
import torch
import torch.nn.functional as F


def _w(bits_or_f32):
    a = np.asarray(bits_or_f32)
    if a.dtype == np.uint16:
        a = (a.astype(np.uint32) << 16).view(np.float32)
    return torch.tensor(a.astype(np.float64))


def bf16_input(x_nhwc_f32):
    t = torch.tensor(np.asarray(x_nhwc_f32, np.float32)).to(torch.bfloat16).to(torch.float64)
    return t.permute(2, 0, 1)[None]          # 1,C,H,W


def conv(x, W, name, stride):
    w = _w(W[name + ".w"]).permute(0, 3, 1, 2)   # Co,Ci,k,k
    return F.conv2d(x, w, _w(W[name + ".b"]), stride=stride, padding=w.shape[-1] // 2)


def shortcut_a(x, c_out):
    sub = x[:, :, ::2, ::2]
    p = (c_out - x.shape[1]) // 2
    return F.pad(sub, (0, 0, 0, 0, p, c_out - x.shape[1] - p))


def block(x, W, i, per_stage):
    s = (i - 1) // per_stage
    first = (i - 1) % per_stage == 0
    stride = 2 if (s > 0 and first) else 1
    c_out = (16, 32, 64)[s]
    t = F.relu(conv(x, W, f"b{i}.c1", stride))
    sc = x if stride == 1 else shortcut_a(x, c_out)
    return F.relu(conv(t, W, f"b{i}.c2", 1) + sc)


def head(x, W, name):
    g = x.mean(dim=(2, 3))[0]
    return _w(W[name + ".w"]) @ g + _w(W[name + ".b"])


def static_resnet(x_f32, W, per_stage, upto=None, exec_blocks=None):
    """Run stem + blocks 1..upto; blocks not in exec_blocks take the shortcut only."""
    x = bf16_input(x_f32)
    x = F.relu(conv(x, W, "stem", 1))
    n = upto or 3 * per_stage
    for i in range(1, n + 1):
        if exec_blocks is None or i in exec_blocks:
            x = block(x, W, i, per_stage)
        else:
            s = (i - 1) // per_stage
            if s > 0 and (i - 1) % per_stage == 0:
                x = shortcut_a(x, (16, 32, 64)[s])
    return x
