"""Benchmark: batched dynamic-NN inference (DyCL, arXiv 2307.04963) on B200.

Headline workload (BASELINE.json configs[4], the largest configuration and the one its
multi-GPU metric "samples/sec at 1/2/4/8 B200" is sharded on): early-exit ResNet-50 v1.5 on
synthetic 224x224x3 inputs, exits after stages 1/2/3 + final head (1000 classes), tau = 0.9,
calibrated heads (workloads/calib/cfg5.json), GLOBAL batch 65536 sharded over the ranks
(rank r takes samples [r*B/G, (r+1)*B/G): strong scaling), each rank's shard resident in
HBM and processed in chunks of 2048 through the C ABI (dycl_run).  One step = one full
pass of the hot path (input cast, every sub-network, predicates, compaction, gathers,
scatters) over the whole global batch.  With G > 1 the survivors of exit 0 are rebalanced
across ranks inside dycl_run over NCCL (dycl_set_comm; --no-rebalance disables).

  python bench.py [--gpus N --steps K --warmup W] [--config 2]   # our arm (default config 5)
  python bench.py --impl reference ...                          # the CPU oracle arm
  torchrun --nproc-per-node N bench.py --gpus N ...             # N > 1: one rank per GPU

Other configs (--config 1..4) are secondary lines: per-GPU batches as BASELINE.json states
them (weak scaling).  Timing = max over ranks of the per-rank device time (CUDA events).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "dynamic-inference samples/sec"
UNIT = "samples/s"
DEFAULT_CONFIG = 5
GLOBAL_BATCH_CONFIGS = {5}         # BASELINE configs[4]: "batch 65536 sharded over 1/2/4/8 B200"
CHUNK = {5: 2048}                  # per-dycl_run chunk (graph finalised for this many rows)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p["bf16_tflops_sustained"], "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def shard(B, ws, rank):
    """Rank r's contiguous slice [r*B/G, (r+1)*B/G) of a global batch."""
    return rank * B // ws, (rank + 1) * B // ws


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = f"/tmp/dycl_clocks_{os.getpid()}.csv"

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 9:
                    continue
                sm.append(float(f[1]))
                mx.append(float(f[2]))
                for n, v in zip(names, f[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
        except Exception:
            return None
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


WORKLOADS = {
    1: "cfg1: tiny early-exit MLP, 3 blocks width 64, 2 exit heads + final, tau=0.9, batch 32 random fp32 inputs",
    2: "cfg2: ShallowDeep-style early-exit ResNet-56, synthetic 32x32x3 CIFAR-shaped inputs, 4 ICs after blocks "
       "5/11/16/22 + final head, tau=0.9, calibrated heads, batch 4096 per GPU",
    3: "cfg3: SkipNet-style gated ResNet-38, 17 feed-forward gates, synthetic 32x32x3, batch 8192 per GPU",
    4: "cfg4: 6+6 post-LN Transformer d=512, greedy decode with per-sequence EOS / max-len 64 loop guard, "
       "batch 1024 random-token sequences (src len 64) per GPU",
    5: "cfg5: early-exit ResNet-50 v1.5, synthetic 224x224x3, exits after stages 1/2/3 + final (1000 classes), "
       "tau=0.9, global batch 65536 sharded over the GPUs (inputs resident in HBM, chunks of 2048 per dycl_run)",
}
BATCHES = {1: 32, 2: 4096, 3: 8192, 4: 1024, 5: 65536}
CAP_WORKLOAD = ("image-captioning En-Decoder (SURVEY 8(f)4): CIFAR ResNet-38 trunk encoder (8x8x64 annotation "
                "vectors), soft-attention LSTM decoder (hidden 256, vocab 4096), greedy with EOS / max-len 32 guard, "
                "batch 1024 synthetic 32x32x3 images per GPU")
RNN_NOTE = " -- variant: recurrent LSTM gates (SkipNet RNN gate, Table 3 ID 5), hidden 10, shared across the 17 gates"
KERNEL_NAMES = {
    "block": "k_block_fused (a1: 1-8 whole residual blocks per sample, SMEM-resident, row-tap tcgen05 convs)",
    "conv": "a1 conv class (k_conv_gemm NHWC TMA-im2col GEMM / k_conv_tma / k_gemm_tma on tcgen05, fused epilogue)",
    "gemm": "k_gemm_tma (a7/a8 decoder + encoder projections, FFN, LM head on tcgen05)",
    "attn": "a7/a8 attention (decode KV streaming / encoder)",
}


def oracle_sample(cfg, n, start=0, rnn=False, caption=False):
    """The oracle (as it stands, mirror mode, all host cores) on n seeded samples of config cfg.
    Returns (samples/s, cores, seconds, description)."""
    import oracle as O
    import workloads as wl
    from oracle import programs as prg
    cores = len(os.sched_getaffinity(0))
    if caption:
        from concurrent.futures import ThreadPoolExecutor
        from oracle import caption as C
        P = prg.prepare(wl.caption_weights())
        X = wl.image_inputs(wl.INPUT_SEED, start, n)
        t0 = time.perf_counter()
        with ThreadPoolExecutor(cores) as ex:
            list(ex.map(lambda i: C.caption(X[i], P, wl.CAP, "mirror"), range(n)))
        dt = time.perf_counter() - t0
        return n / dt, cores, dt, (f"{n} captioning images (seeded inputs {start}..{start + n - 1}), per-image fp64 "
                                   f"encoder + greedy decode, mirror mode")
    if cfg == 4:
        from concurrent.futures import ThreadPoolExecutor
        from oracle import seq2seq as S
        P = S.prepare_s2s(wl.seq2seq_weights())
        src = wl.token_inputs(wl.INPUT_SEED, start, n)
        t0 = time.perf_counter()
        with ThreadPoolExecutor(cores) as ex:
            list(ex.map(lambda i: S.greedy_decode(src[i], P, wl.S2S, "mirror"), range(n)))
        dt = time.perf_counter() - t0
        return n / dt, cores, dt, (f"{n} cfg4 sequences (seeded tokens {start}..{start + n - 1}), per-sequence fp64 "
                                   f"greedy decode, mirror mode")
    W = {1: wl.mlp_weights, 2: wl.sdn_r56_weights, 3: wl.skipnet_r38_weights, 5: wl.resnet50_ee_weights}[cfg]()
    program = O.PROGRAMS[cfg]
    if rnn and cfg == 3:
        W, program = wl.skipnet_rnn_r38_weights(), O.skipnet_rnn_resnet38
    P = prg.prepare(W)
    X = (wl.mlp_inputs(wl.INPUT_SEED, start, n) if cfg == 1 else
         wl.image_inputs(wl.INPUT_SEED, start, n, hw=224 if cfg == 5 else 32))
    t0 = time.perf_counter()
    O.run_batch(program, X, P, "mirror", threads=cores)
    dt = time.perf_counter() - t0
    return n / dt, cores, dt, (f"{n} cfg{cfg} samples (seeded inputs {start}..{start + n - 1}), per-sample fp64 "
                               f"interpreter, mirror mode")


REF_SAMPLES = {1: 4096, 2: 32, 3: 32, 4: 4, 5: 8}


def run_reference(args):
    """The base contract's reference arm for this tier: the CPU oracle timed as it stands on the
    host cores, each step a bounded sample of the same workload (rank 0 only)."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    per_step = args.ref_samples or REF_SAMPLES[args.config]
    times = []
    what = ""
    cores = len(os.sched_getaffinity(0))
    for i in range(args.warmup + args.steps):
        _, cores, dt, what = oracle_sample(args.config, per_step, start=i * per_step, rnn=args.rnn_gates,
                                           caption=args.caption)
        if i >= args.warmup:
            times.append(dt)
    tot = sum(times)
    value = per_step * args.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "strong" if args.config in GLOBAL_BATCH_CONFIGS else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.config] + (RNN_NOTE if args.rnn_gates and args.config == 3 else ""),
                   "samples_per_step": per_step},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"per step: {what}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


class ImageJob:
    """configs 1/2/3/5: one step = dycl_run over every chunk of this rank's samples."""

    def __init__(self, cfg, rank, ws, dev, torch, rebalance, rnn=False):
        import workloads as wl
        from paper_2307_04963_b200 import programs as P
        self.cfg, self.torch = cfg, torch
        if cfg in GLOBAL_BATCH_CONFIGS:
            g0, g1 = shard(BATCHES[cfg], ws, rank)
            self.B = g1 - g0
            per_rank_max = max(shard(BATCHES[cfg], ws, r)[1] - shard(BATCHES[cfg], ws, r)[0] for r in range(ws))
        else:
            g0, self.B = rank * BATCHES[cfg], BATCHES[cfg]
            per_rank_max = self.B
        self.g0 = g0
        chunk = CHUNK.get(cfg, per_rank_max)
        # the same number of chunks on every rank (rebalancing runs them in lock step)
        self.n_chunks = max(1, (per_rank_max + chunk - 1) // chunk)
        self.bounds = [self.B * i // self.n_chunks for i in range(self.n_chunks + 1)]
        self.chunk = max(b - a for a, b in zip(self.bounds, self.bounds[1:]))
        W = {1: wl.mlp_weights, 2: wl.sdn_r56_weights, 3: wl.skipnet_r38_weights, 5: wl.resnet50_ee_weights}[cfg]()
        build = P.BUILDERS[cfg]
        if rnn and cfg == 3:
            W, build = wl.skipnet_rnn_r38_weights(), P.build_skipnet_rnn_resnet38
        self.model = build(W, (per_rank_max + self.n_chunks - 1) // self.n_chunks + 1, device=dev.index or 0)
        self.rebalance = False
        if rebalance and ws > 1:
            from paper_2307_04963_b200 import dist as DI
            DI.attach(self.model, rank, ws)
            if rebalance == "device":
                from paper_2307_04963_b200 import dycl as D
                D.dycl_set_rebalance_mode(self.model.g, D.DYCL_REBALANCE_MODE_DEVICE)
            self.rebalance = True
        if cfg == 1:
            X = torch.from_numpy(wl.mlp_inputs(wl.INPUT_SEED, g0, self.B)).to(dev)
        elif cfg == 5:
            X = wl.image_inputs_torch(wl.INPUT_SEED, g0, self.B, hw=224, device=dev)
        else:
            X = torch.from_numpy(wl.image_inputs(wl.INPUT_SEED, g0, self.B)).to(dev)
        self.x = X
        K = self.model.K
        self.logits = torch.empty((self.B, K), device=dev)
        self.path = torch.empty(self.B, dtype=torch.int32, device=dev)
        self.g = self.model.g
        self.h2d = int(X.numel() * 4)
        self.d2h = int(self.B * (K * 4 + 4))

    def chunks(self):
        return zip(self.bounds, self.bounds[1:])

    def step(self, stream, after_chunk=None):
        for c0, c1 in self.chunks():
            self.model.run(self.x[c0:c1], self.logits[c0:c1], self.path[c0:c1], stream=stream,
                           global_offset=self.g0 + c0)
            if after_chunk:
                after_chunk()

    def host_setup(self):
        torch = self.torch
        self.xh = self.x.cpu().pin_memory()
        self.lh = torch.empty(tuple(self.logits.shape), dtype=torch.float32).pin_memory()
        self.ph = torch.empty(self.B, dtype=torch.int32).pin_memory()

    def step_host(self, stream):
        # one public call for the rank's whole shard: the library streams it through in
        # max_batch-row sub-chunks with the copies of sub-chunk k +- 1 under the run of k
        self.model.run_host(self.xh, self.lh, self.ph, stream=stream, global_offset=self.g0)

    def check_host(self):
        return bool(np.array_equal(self.ph.numpy(), self.path.cpu().numpy()))

    def hist(self):
        p = self.path.cpu().numpy()
        return np.bincount(p, minlength=5).tolist() if self.cfg != 3 else \
            {"mean_blocks_executed": float(np.mean([bin(int(v)).count("1") for v in p]) + 1)}


class S2SJob:
    """config 4: one step = encoder + guarded greedy decode of the per-rank batch."""

    def __init__(self, cfg, rank, ws, dev, torch, rebalance, rnn=False):
        import workloads as wl
        from paper_2307_04963_b200 import programs as P
        self.cfg, self.torch = cfg, torch
        self.B = BATCHES[4]
        self.n_chunks = 1
        self.rebalance = False
        c = wl.S2S
        self.model = P.build_seq2seq(wl.seq2seq_weights(), c, self.B, device=dev.index or 0)
        self.g = None
        src = wl.token_inputs(wl.INPUT_SEED, rank * self.B, self.B)
        self.src = torch.from_numpy(src).to(dev)
        self.tok = torch.empty((self.B, c["max_len"]), dtype=torch.int32, device=dev)
        self.len = torch.empty(self.B, dtype=torch.int32, device=dev)
        self.h2d = int(src.nbytes)
        self.d2h = int(self.B * (c["max_len"] + 1) * 4)

    def step(self, stream, after_chunk=None):
        self.model.run(self.src, self.tok, self.len, stream=stream)
        if after_chunk:
            after_chunk()

    def host_setup(self):
        torch = self.torch
        self.sh = self.src.cpu().pin_memory()
        self.th = torch.empty(tuple(self.tok.shape), dtype=torch.int32).pin_memory()
        self.lh = torch.empty(self.B, dtype=torch.int32).pin_memory()

    def step_host(self, stream):
        self.model.run_host(self.sh, self.th, self.lh, stream=stream)

    def check_host(self):
        return bool(np.array_equal(self.lh.numpy(), self.len.cpu().numpy()))

    def hist(self):
        ln = self.len.cpu().numpy()
        return {"mean_length": float(ln.mean()), "tokens": int(ln.sum())}


class CapJob:
    """--caption: the image-captioning En-Decoder (reading R20): one step = the CNN
    encoder graph + the guarded soft-attention LSTM decode of the per-rank batch of 1024 images."""

    def __init__(self, cfg, rank, ws, dev, torch, rebalance, rnn=False):
        import workloads as wl
        from paper_2307_04963_b200 import programs as P
        self.cfg, self.torch = cfg, torch
        self.B = 1024
        self.n_chunks = 1
        self.rebalance = False
        c = wl.CAP
        self.model = P.build_caption(wl.caption_weights(), c, self.B, device=dev.index or 0)
        self.g = None
        X = wl.image_inputs(wl.INPUT_SEED, rank * self.B, self.B)
        self.x = torch.from_numpy(X).to(dev)
        self.tok = torch.empty((self.B, c["max_len"]), dtype=torch.int32, device=dev)
        self.len = torch.empty(self.B, dtype=torch.int32, device=dev)
        self.feats = torch.empty((self.B, c["L"], c["D"]), dtype=torch.int16, device=dev)
        self.h2d = int(X.nbytes)
        self.d2h = int(self.B * (c["max_len"] + 1) * 4)

    def step(self, stream, after_chunk=None):
        self.model.run(self.x, self.tok, self.len, stream=stream, features=self.feats)
        if after_chunk:
            after_chunk()

    def host_setup(self):
        torch = self.torch
        self.xh = self.x.cpu().pin_memory()
        self.th = torch.empty(tuple(self.tok.shape), dtype=torch.int32).pin_memory()
        self.lh = torch.empty(self.B, dtype=torch.int32).pin_memory()

    def step_host(self, stream):
        # the public call chain with host buffers: H2D of the images, encoder + decoder, D2H
        self.x.copy_(self.xh, non_blocking=True)
        self.model.run(self.x, self.tok, self.len, stream=stream, features=self.feats)
        self.th.copy_(self.tok, non_blocking=True)
        self.lh.copy_(self.len, non_blocking=True)
        self.torch.cuda.current_stream().synchronize()

    def check_host(self):
        return bool(np.array_equal(self.lh.numpy(), self.len.cpu().numpy()))

    def hist(self):
        ln = self.len.cpu().numpy()
        return {"mean_length": float(ln.mean()), "tokens": int(ln.sum())}


def _traffic(cfg, kind):
    """ncu DRAM bytes per launch of the dominant kernel class (profiles/r02_traffic.json, one
    `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum` capture of one step / chunk)."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "r02_traffic.json")))
        return t[f"cfg{cfg}"][kind]["dram_bytes_per_launch"]
    except Exception:
        return None


def run_dycl(args):
    import torch
    from paper_2307_04963_b200 import dycl as D

    ws, rank, local = _dist()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    stream = torch.cuda.current_stream()
    job_cls = CapJob if args.caption else S2SJob if args.config == 4 else ImageJob
    job = job_cls(args.config, rank, ws, dev, torch, False if args.no_rebalance else args.rebalance_mode,
                  rnn=args.rnn_gates)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > L2 (126 MB)

    for _ in range(args.warmup):
        job.step(stream)
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()

    # Pass 1 (the number): K timed steps, one CUDA-event pair per step on the launch stream.
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = ClockSampler(local)
    clocks.start()
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.zero_()                          # evict L2 between timed steps (not timed)
        ev[i][0].record(stream)
        job.step(stream)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    # Pass 2 (the roofline): the same K steps again with per-launch CUDA events recorded by
    # libdycl on the launch stream around every kernel, read back after every chunk (kept out
    # of pass 1: the event pairs perturb the step time).
    kind_tot = {}                              # kind -> [ms, bytes, flops, launches, records]
    n_prof = [0]
    if args.caption:
        prof_read = lambda: []                           # noqa: E731  (no per-launch profiling here)
    elif job.g is not None:
        D.dycl_set_profiling(job.g, 1)
        prof_read = lambda: D.dycl_profile_read(job.g)   # noqa: E731
    else:
        D.dycl_s2s_set_profiling(job.model.h, 1)
        prof_read = lambda: D.dycl_s2s_profile_read(job.model.h)   # noqa: E731

    def collect():
        for p in prof_read():                  # syncs the stream
            n_prof[0] += 1
            t = kind_tot.setdefault(p["kind"], [0.0, 0.0, 0.0, 0, []])
            t[0] += p["ms"]
            t[1] += p["bytes"]
            t[2] += p["flops"]
            t[3] += 1
            t[4].append((p["ms"], p["bytes"], p["flops"]))

    for i in range(args.steps):
        flush.zero_()
        job.step(stream, after_chunk=collect)
    torch.cuda.synchronize()
    if args.caption:
        launches = (D.dycl_cap_launches(job.model.h) + D.dycl_launches_per_run(job.model.enc.g)) * args.steps
    elif job.g is not None:
        D.dycl_set_profiling(job.g, 0)
        launches = n_prof[0]                   # this library's kernels in K steps (profiled pass)
    else:
        D.dycl_s2s_set_profiling(job.model.h, 0)
        launches = n_prof[0]
    kind_ms = {k: v[0] for k, v in kind_tot.items()}
    hist = job.hist()

    # e2e: the public host-buffer call (pinned buffers; H2D + run + D2H each step)
    job.host_setup()
    job.step_host(stream)
    torch.cuda.synchronize()
    e2e_ms = 0.0
    for i in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        job.step_host(stream)
        e2e_ms += (time.perf_counter() - t0) * 1e3
    assert job.check_host(), "host-buffer run disagrees with device run"

    t = torch.tensor([total_ms, e2e_ms], dtype=torch.float64, device=dev)
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.barrier()
    total_ms, e2e_ms = float(t[0]), float(t[1])
    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        return

    hbm, tf_burst, tf_sus, peak_src = _peaks()
    global_samples = (1024 * ws if args.caption else
                      BATCHES[args.config] if args.config in GLOBAL_BATCH_CONFIGS else BATCHES[args.config] * ws)
    value = global_samples * args.steps / (total_ms / 1e3)
    # a step of >= 100 ms keeps the tensor pipe busy long enough to reach the sustained
    # (power-limited) clock: the sustained peak applies; shorter steps: the burst peak
    long_step = total_ms / args.steps >= 100.0
    tf_peak = tf_sus if long_step else tf_burst
    roof = None
    step_prof_ms = sum(kind_ms.values())
    if kind_tot:
        dom = max(kind_tot, key=lambda k: kind_tot[k][0])
        ms_, by_, fl_, n_, recs = kind_tot[dom]
        gbs = by_ / (ms_ / 1e3) / 1e9
        tfl = fl_ / (ms_ / 1e3) / 1e12
        # per-launch roofline: ideal = max(FLOPs / tensor peak, bytes / HBM peak)
        split = {"tensor": [0.0, 0.0], "hbm": [0.0, 0.0]}
        for lm, lb, lf in recs:
            it, ib = lf / (tf_peak * 1e12) * 1e3, lb / (hbm * 1e9) * 1e3
            k = "tensor" if it > ib else "hbm"
            split[k][0] += max(it, ib)
            split[k][1] += lm
        roof_eff = (split["tensor"][0] + split["hbm"][0]) / ms_ if ms_ else None
        tensor_bound = split["tensor"][1] > split["hbm"][1]
        traffic = _traffic(args.config, dom)
        if tensor_bound:
            roof = {"kernel": KERNEL_NAMES.get(dom, dom), "bound": "tensor", "achieved": tfl, "peak": tf_peak,
                    "unit": "TFLOP/s", "frac": tfl / tf_peak, "traffic": traffic,
                    "peak_source": peak_src + (" bf16 sustained (step >= 100 ms)" if long_step else " bf16 burst"),
                    "frac_of_burst": tfl / tf_burst, "frac_of_sustained": tfl / tf_sus, "hbm_GBps": gbs}
        else:
            roof = {"kernel": KERNEL_NAMES.get(dom, dom), "bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s",
                    "frac": gbs / hbm, "traffic": traffic, "peak_source": peak_src,
                    "tensor_tflops": tfl, "tensor_frac_of_burst": tfl / tf_burst}
        roof.update({"roofline_efficiency": roof_eff,
                     "launch_split": {k: {"ms_per_step": v[1] / args.steps,
                                          "frac_of_own_roofline": v[0] / v[1] if v[1] else None}
                                      for k, v in split.items()},
                     "share_of_step": ms_ / step_prof_ms if step_prof_ms else None,
                     "algorithmic_bytes_per_launch": by_ / max(n_, 1),
                     "algorithmic_flops_per_launch": fl_ / max(n_, 1),
                     "avg_launch_ms": ms_ / max(n_, 1),
                     "launches_per_step": n_ // max(args.steps, 1),
                     "measured": "per-launch CUDA events (libdycl profiling) on the launch stream over a second "
                                 "pass of the same K steps (every chunk); achieved = algorithmic bytes (or FLOPs) "
                                 "/ kernel time; traffic = ncu DRAM read+write bytes per launch "
                                 "(profiles/r02_traffic.json)",
                     "classes": {k: {"ms_per_step": v[0] / args.steps, "share": v[0] / step_prof_ms,
                                     "GBps": v[1] / (v[0] / 1e3) / 1e9 if v[0] else 0.0,
                                     "TFLOPs": v[2] / (v[0] / 1e3) / 1e12 if v[0] else 0.0}
                                 for k, v in sorted(kind_tot.items(), key=lambda kv: -kv[1][0])}})
    strong = args.config in GLOBAL_BATCH_CONFIGS
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "ms_per_step_std": float(np.std(step_ms)),
        "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic",
        "config": {"workload": (CAP_WORKLOAD if args.caption else
                                WORKLOADS[args.config] + (RNN_NOTE if args.rnn_gates and args.config == 3 else "")),
                   "global_batch": global_samples,
                   "batch_per_gpu": job.B, "chunks_per_gpu": job.n_chunks,
                   "precision": "bf16 tensor-core operands, fp32 accumulate, fp32 residual stream",
                   "l2": "flushed (256 MB write) before every timed step, flush not timed; inputs > L2",
                   "parallelism": (f"dp{ws}: contiguous shards of the global batch" if strong else
                                   f"dp{ws}: independent per-GPU batches") +
                                  (f"; survivors rebalanced after every exit inside dycl_run ({args.rebalance_mode}-initiated)"
                                   if job.rebalance
                                   else "; no collective on the data path"),
                   "decisions_rank0": hist},
        "clocks": clk,
        "e2e": {"value": global_samples * args.steps / (e2e_ms / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": job.h2d, "d2h_bytes_per_step": job.d2h},
        "gpu_launches": launches,
        "roofline": roof,
        "kernel_ms_per_step": {k: v / args.steps for k, v in sorted(kind_ms.items(), key=lambda kv: -kv[1])},
    }
    if args.config == 4 or args.caption:
        line["tokens_per_s"] = hist["tokens"] * ws * args.steps / (total_ms / 1e3)
    if ws == 1 and not args.no_cpu_baseline:
        n_cpu = args.cpu_samples or (64 if args.caption else {1: 4096, 2: 4096, 3: 2048, 4: 48, 5: 64}[args.config])
        rate, cores, dt, what = oracle_sample(args.config, n_cpu, rnn=args.rnn_gates, caption=args.caption)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle",
                                "sample": f"{what}, {dt:.1f} s wall"}
    print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="default: 10 for config 5, 50 otherwise")
    ap.add_argument("--warmup", type=int, default=None, help="default: 3 for config 5, 5 otherwise")
    ap.add_argument("--impl", default="dycl", choices=["dycl", "reference"])
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG, choices=[1, 2, 3, 4, 5],
                    help="BASELINE.json config (default 5: the largest, global batch 65536 sharded over the GPUs)")
    ap.add_argument("--cpu-samples", type=int, default=None)
    ap.add_argument("--ref-samples", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-rebalance", action="store_true", help="N > 1: no survivor rebalancing")
    ap.add_argument("--rebalance-mode", default="host", choices=["host", "device"],
                    help="N > 1: survivor exchange via the host plan + NCCL send/recv, or device-initiated "
                         "through NCCL symmetric windows (SURVEY 8(f)1)")
    ap.add_argument("--caption", action="store_true",
                    help="the image-captioning En-Decoder (SURVEY 8(f)4): CNN encoder + soft-attention LSTM decoder")
    ap.add_argument("--rnn-gates", action="store_true",
                    help="config 3 with SkipNet's recurrent (LSTM) gates (SURVEY 8(f)3, Table 3 ID 5)")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 10 if args.config == 5 else 50
    if args.warmup is None:
        args.warmup = 3 if args.config == 5 else 5
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_dycl(args)


if __name__ == "__main__":
    main()
