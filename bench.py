"""Benchmark: batched dynamic-NN inference (DyCL, arXiv 2307.04963) on B200.

Workload (BASELINE.json configs[1], the configuration its metric is quoted on):
ShallowDeep-style early-exit ResNet-56 on synthetic 32x32x3 CIFAR-shaped inputs,
batch 4096 per GPU, 4 internal classifiers + final head, tau = 0.9, calibrated
heads (workloads/calib/cfg2.json).  One step = one full pass of the hot path
(input cast, every sub-network, predicates, compaction, gathers, scatters) over
one batch, through the C ABI (dycl_run).

  python bench.py [--gpus N --steps K --warmup W]            # our arm
  python bench.py --impl reference ...                        # the CPU oracle arm
  torchrun --nproc-per-node N bench.py --gpus N ...           # N > 1: one rank per GPU

Multi-GPU: samples are independent (Eq. 2 is per-x), so each rank processes its
own 4096-sample slice of the global batch (weak scaling) with no collective on
the data path; timing = max over ranks of the per-rank device time.
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
BATCH = 4096
WORKLOAD = ("cfg2: ShallowDeep-style early-exit ResNet-56, synthetic 32x32x3 CIFAR-shaped inputs, "
            "4 ICs after blocks 5/11/16/22 + final head, tau=0.9, calibrated heads")


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p["bf16_tflops_sustained"], "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


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


def cpu_oracle_rate(n_samples: int, seed_offset: int = 0):
    """The oracle (as it stands) on this host's cores: per-sample interpreter, mirror mode."""
    import oracle as O
    import workloads as wl
    from oracle import programs as prg
    P = prg.prepare(wl.sdn_r56_weights())
    X = wl.image_inputs(wl.INPUT_SEED, seed_offset, n_samples)
    cores = len(os.sched_getaffinity(0))
    t0 = time.perf_counter()
    O.run_batch(O.sdn_resnet56, X, P, "mirror", threads=cores)
    dt = time.perf_counter() - t0
    return n_samples / dt, cores, dt


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    per_step = args.ref_samples
    times = []
    cores = len(os.sched_getaffinity(0))
    for i in range(args.warmup + args.steps):
        rate, cores, dt = cpu_oracle_rate(per_step, seed_offset=i * per_step)
        if i >= args.warmup:
            times.append(dt)
    tot = sum(times)
    value = per_step * args.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": WORKLOAD, "samples_per_step": per_step},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{per_step} samples of cfg2 per step (seeded inputs), per-sample fp64 interpreter"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


WORKLOADS = {
    1: "cfg1: tiny early-exit MLP, 3 blocks width 64, 2 exit heads + final, tau=0.9, batch 32 random fp32 inputs",
    2: WORKLOAD,
    3: "cfg3: SkipNet-style gated ResNet-38, 17 feed-forward gates, synthetic 32x32x3, batch 8192",
    4: "cfg4: 6+6 post-LN Transformer d=512, greedy decode with per-sequence EOS / max-len 64 loop guard, "
       "batch 1024 random-token sequences (src len 64)",
    5: "cfg5: early-exit ResNet-50 v1.5, synthetic 224x224x3, exits after stages 1/2/3 + final, batch 65536 per GPU "
       "(processed in chunks of 2048, all inputs resident in HBM)",
}
BATCHES = {1: 32, 2: 4096, 3: 8192, 4: 1024, 5: 65536}


class ImageJob:
    """configs 1/2/3/5: one step = dycl_run over every chunk of the per-rank batch."""

    def __init__(self, cfg, rank, dev, torch):
        import workloads as wl
        from paper_2307_04963_b200 import programs as P
        self.cfg, self.torch = cfg, torch
        self.B = BATCHES[cfg]
        self.chunk = 2048 if cfg == 5 else self.B
        W = {1: wl.mlp_weights, 2: wl.sdn_r56_weights, 3: wl.skipnet_r38_weights, 5: wl.resnet50_ee_weights}[cfg]()
        self.model = P.BUILDERS[cfg](W, self.chunk, device=dev.index or 0)
        g0 = rank * self.B
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

    def step(self, stream):
        for c0 in range(0, self.B, self.chunk):
            c1 = min(self.B, c0 + self.chunk)
            self.model.run(self.x[c0:c1], self.logits[c0:c1], self.path[c0:c1], stream=stream)

    def host_setup(self):
        torch = self.torch
        self.xh = self.x.cpu().pin_memory()
        self.lh = torch.empty(tuple(self.logits.shape), dtype=torch.float32).pin_memory()
        self.ph = torch.empty(self.B, dtype=torch.int32).pin_memory()

    def step_host(self, stream):
        for c0 in range(0, self.B, self.chunk):
            c1 = min(self.B, c0 + self.chunk)
            self.model.run_host(self.xh[c0:c1], self.lh[c0:c1], self.ph[c0:c1], stream=stream)

    def check_host(self):
        return bool(np.array_equal(self.ph.numpy(), self.path.cpu().numpy()))

    def hist(self):
        p = self.path.cpu().numpy()
        return np.bincount(p, minlength=5).tolist() if self.cfg != 3 else \
            {"mean_blocks_executed": float(np.mean([bin(int(v)).count("1") for v in p]) + 1)}


class S2SJob:
    """config 4: one step = encoder + guarded greedy decode of the per-rank batch."""

    def __init__(self, cfg, rank, dev, torch):
        import workloads as wl
        from paper_2307_04963_b200 import programs as P
        self.cfg, self.torch = cfg, torch
        self.B = BATCHES[4]
        c = wl.S2S
        self.model = P.build_seq2seq(wl.seq2seq_weights(), c, self.B, device=dev.index or 0)
        self.g = None
        src = wl.token_inputs(wl.INPUT_SEED, rank * self.B, self.B)
        self.src = torch.from_numpy(src).to(dev)
        self.tok = torch.empty((self.B, c["max_len"]), dtype=torch.int32, device=dev)
        self.len = torch.empty(self.B, dtype=torch.int32, device=dev)
        self.h2d = int(src.nbytes)
        self.d2h = int(self.B * (c["max_len"] + 1) * 4)

    def step(self, stream):
        self.model.run(self.src, self.tok, self.len, stream=stream)

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
    job = (S2SJob if args.config == 4 else ImageJob)(args.config, rank, dev, torch)
    B = job.B
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
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    # Pass 2 (the roofline): the same K steps again with per-launch CUDA events recorded by
    # libdycl on the launch stream around every kernel (kept out of pass 1: ~80 event pairs
    # per step perturb the step time).
    # per-kind totals: ms, algorithmic bytes, algorithmic flops, launches
    kind_tot = {}
    launches = 0
    if job.g is not None:
        D.dycl_set_profiling(job.g, 1)
        prof_read = lambda: D.dycl_profile_read(job.g)   # noqa: E731
    else:
        D.dycl_s2s_set_profiling(job.model.h, 1)
        prof_read = lambda: D.dycl_s2s_profile_read(job.model.h)   # noqa: E731
    for i in range(args.steps):
        flush.zero_()
        job.step(stream)     # profiling records the last chunk's launches; chunks are identical in shape
        for p in prof_read():    # syncs the stream
            t = kind_tot.setdefault(p["kind"], [0.0, 0.0, 0.0, 0, []])
            t[0] += p["ms"]
            t[1] += p["bytes"]
            t[2] += p["flops"]
            t[3] += 1
            t[4].append((p["ms"], p["bytes"], p["flops"]))
    torch.cuda.synchronize()
    if job.g is not None:
        D.dycl_set_profiling(job.g, 0)
        launches = D.dycl_launches_per_run(job.g) * args.steps * ((B + job.chunk - 1) // job.chunk)
    else:
        D.dycl_s2s_set_profiling(job.model.h, 0)
        launches = D.dycl_s2s_launches(job.model.h) * args.steps
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
    value = B * ws * args.steps / (total_ms / 1e3)
    roof = None
    step_prof_ms = sum(kind_ms.values())
    if kind_tot:
        # the dominant kernel class of the step (largest share of the per-launch event time)
        dom = max(kind_tot, key=lambda k: kind_tot[k][0])
        ms_, by_, fl_, n_, recs = kind_tot[dom]
        gbs = by_ / (ms_ / 1e3) / 1e9
        tfl = fl_ / (ms_ / 1e3) / 1e12
        # per-launch roofline: ideal = max(FLOPs / tensor peak, bytes / HBM peak); a launch is
        # tensor- or HBM-bound by which term wins; efficiency = sum(ideal) / sum(measured)
        split = {"tensor": [0.0, 0.0], "hbm": [0.0, 0.0]}
        for lm, lb, lf in recs:
            it, ib = lf / (tf_sus * 1e12) * 1e3, lb / (hbm * 1e9) * 1e3
            k = "tensor" if it > ib else "hbm"
            split[k][0] += max(it, ib)
            split[k][1] += lm
        roof_eff = (split["tensor"][0] + split["hbm"][0]) / ms_ if ms_ else None
        names = {
            "block": "k_block_fused (a1: 1-8 whole residual blocks per sample, SMEM-resident, row-tap tcgen05 convs)",
            "conv": "a1 conv class (k_conv_gemm NHWC im2col GEMM / k_conv_tma / k_gemm_tma on tcgen05, fused epilogue)",
            "gemm": "k_gemm_tma (a7/a8 decoder + encoder projections, FFN, LM head on tcgen05)",
            "attn": "k_attn_decoder (a7 decode attention, KV-cache streaming)",
        }
        tensor_bound = split["tensor"][1] > split["hbm"][1]   # the bound that covers most of the class's time
        if tensor_bound:
            roof = {"kernel": names.get(dom, dom), "bound": "tensor", "achieved": tfl, "peak": tf_sus,
                    "unit": "TFLOP/s", "frac": tfl / tf_sus, "traffic": None,
                    "peak_source": peak_src + " bf16 sustained", "hbm_GBps": gbs}
        else:
            traffic = None
            tpath = os.path.join(ROOT, "profiles", "block_traffic.json")
            if dom == "block" and args.config == 2 and os.path.exists(tpath):
                try:
                    traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
                except Exception:
                    traffic = None
            roof = {"kernel": names.get(dom, dom), "bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s",
                    "frac": gbs / hbm, "traffic": traffic, "peak_source": peak_src,
                    "tensor_tflops": tfl, "tensor_frac_of_sustained": tfl / tf_sus}
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
                                 "pass of the same K steps; achieved = algorithmic bytes (or FLOPs) / kernel time",
                     "classes": {k: {"ms_per_step": v[0] / args.steps, "share": v[0] / step_prof_ms,
                                     "GBps": v[1] / (v[0] / 1e3) / 1e9 if v[0] else 0.0,
                                     "TFLOPs": v[2] / (v[0] / 1e3) / 1e12 if v[0] else 0.0}
                                 for k, v in sorted(kind_tot.items(), key=lambda kv: -kv[1][0])}})
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.config], "batch_per_gpu": B, "global_batch": B * ws,
                   "precision": "bf16 tensor-core operands, fp32 accumulate, fp32 residual stream",
                   "l2": "flushed (256 MB write) before every timed step, flush not timed",
                   "parallelism": f"dp{ws} (independent shards, no collective)",
                   "decisions_rank0": hist},
        "clocks": clk,
        "e2e": {"value": B * ws * args.steps / (e2e_ms / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": job.h2d, "d2h_bytes_per_step": job.d2h},
        "gpu_launches": launches,
        "roofline": roof,
        "kernel_ms_per_step": {k: v / args.steps for k, v in sorted(kind_ms.items(), key=lambda kv: -kv[1])},
    }
    if args.config == 4:
        line["tokens_per_s"] = hist["tokens"] * ws * args.steps / (total_ms / 1e3)
    if ws == 1 and not args.no_cpu_baseline:
        n_cpu = {1: 4096, 2: args.cpu_samples, 3: 2048, 4: 48, 5: 32}[args.config]
        rate, cores, dt, what = cpu_oracle_rate_cfg(args.config, n_cpu)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle",
                                "sample": f"{what}, {dt:.1f} s wall"}
    print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def cpu_oracle_rate_cfg(cfg, n):
    """The oracle on this host's cores for a bounded sample of config `cfg`."""
    import oracle as O
    import workloads as wl
    from oracle import programs as prg
    cores = len(os.sched_getaffinity(0))
    if cfg == 2:
        rate, cores, dt = cpu_oracle_rate(n)
        return rate, cores, dt, f"{n} cfg2 samples (seeded inputs 0..{n - 1}), per-sample fp64 interpreter, mirror mode"
    if cfg == 4:
        from concurrent.futures import ThreadPoolExecutor
        from oracle import seq2seq as S
        P = S.prepare_s2s(wl.seq2seq_weights())
        src = wl.token_inputs(wl.INPUT_SEED, 0, n)
        t0 = time.perf_counter()
        with ThreadPoolExecutor(cores) as ex:
            list(ex.map(lambda i: S.greedy_decode(src[i], P, wl.S2S, "mirror"), range(n)))
        dt = time.perf_counter() - t0
        return n / dt, cores, dt, f"{n} cfg4 sequences (seeded tokens), per-sequence fp64 greedy decode, mirror mode"
    W = {1: wl.mlp_weights, 3: wl.skipnet_r38_weights, 5: wl.resnet50_ee_weights}[cfg]()
    P = prg.prepare(W)
    X = (wl.mlp_inputs(wl.INPUT_SEED, 0, n) if cfg == 1 else
         wl.image_inputs(wl.INPUT_SEED, 0, n, hw=224 if cfg == 5 else 32))
    t0 = time.perf_counter()
    O.run_batch(O.PROGRAMS[cfg], X, P, "mirror", threads=cores)
    dt = time.perf_counter() - t0
    return n / dt, cores, dt, f"{n} cfg{cfg} samples (seeded inputs), per-sample fp64 interpreter, mirror mode"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="dycl", choices=["dycl", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5],
                    help="BASELINE.json config (default 2: the configuration the metric is quoted on)")
    ap.add_argument("--cpu-samples", type=int, default=4096)
    ap.add_argument("--ref-samples", type=int, default=32)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_dycl(args)


if __name__ == "__main__":
    main()
