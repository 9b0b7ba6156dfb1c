"""RQ3 analog summary: gpurun_out/rq3.jsonl (tools/rq3_ablation.sh) -> profiles/r02_rq3_ablation.json
and a markdown table (stdout) for DESIGN.md."""
import json
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/rq3.jsonl"
L = [json.loads(l) for l in open(src) if l.strip()]
by = {l["ablation"]: l for l in L}
rows = []
for cfg, name in [("c2", "cfg 2 ResNet-56 exits"), ("c3", "cfg 3 SkipNet-38 FF gates"),
                  ("c3r", "cfg 3r SkipNet-38 LSTM gates"), ("c5", "cfg 5 ResNet-50 exits")]:
    on, off = by.get(cfg + "_on"), by.get(cfg + "_off")
    if not on or not off:
        continue

    def moved(l):
        c = l["roofline"]["classes"]
        return sum(v["GBps"] * v["ms_per_step"] / 1e3 for k, v in c.items() if k == "gather")   # GB per step

    r = dict(config=name, ms_off=off["ms_per_step"], ms_on=on["ms_per_step"],
             accelerate_pct=100.0 * (off["ms_per_step"] - on["ms_per_step"]) / off["ms_per_step"],
             copy_GB_off=moved(off), copy_GB_on=moved(on),
             copy_ms_off=off["kernel_ms_per_step"].get("gather", 0.0), copy_ms_on=on["kernel_ms_per_step"].get("gather", 0.0),
             launches_off=off["gpu_launches"] / off["steps"], launches_on=on["gpu_launches"] / on["steps"])
    rows.append(r)
json.dump({"source": "bench.py per config, default vs DYCL_NO_ZERO_COPY=1 DYCL_NO_INPLACE=1 (identity copies "
                     "materialised); ms per step = CUDA-event device time; copy GB = algorithmic bytes of the gather "
                     "kernels (profiled pass)", "rows": rows}, open("profiles/r02_rq3_ablation.json", "w"), indent=1)
print("| config | C_no (ms/step) | C (ms/step) | accelerate | identity-copy bytes off → on | copy kernel ms off → on | launches/step off → on |")
print("|---|---|---|---|---|---|---|")
for r in rows:
    print(f"| {r['config']} | {r['ms_off']:.3f} | {r['ms_on']:.3f} | {r['accelerate_pct']:.1f} % | "
          f"{r['copy_GB_off']:.2f} → {r['copy_GB_on']:.2f} GB | {r['copy_ms_off']:.3f} → {r['copy_ms_on']:.3f} | "
          f"{r['launches_off']:.0f} → {r['launches_on']:.0f} |")
