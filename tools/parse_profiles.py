"""Turn the gpurun_out/ profiling artefacts into committed summaries under profiles/."""
import csv
import json
import os
import sys
from collections import defaultdict

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
tag = sys.argv[2] if len(sys.argv) > 2 else "r01"
os.makedirs("profiles", exist_ok=True)


def rows(path):
    lines = [l for l in open(path) if l.startswith('"')]
    return list(csv.DictReader(lines))


out = {}
# 1. launch list: per-kernel share of one step (ncu: serialised, cold caches)
if os.path.exists(f"{src}/launches.csv"):
    per = defaultdict(float)
    n = defaultdict(int)
    for r in rows(f"{src}/launches.csv"):
        if r["Metric Name"] == "gpu__time_duration.sum":
            k = r["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", "")
            u = r["Metric Unit"]
            v = float(r["Metric Value"].replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0,
                                                             "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1.0)
            per[k] += v
            n[k] += 1
    tot = sum(per.values())
    out["ncu_launch_list"] = {k: {"launches": n[k], "us": round(per[k], 1), "share": round(per[k] / tot, 4)}
                              for k in sorted(per, key=lambda k: -per[k])}
    out["ncu_launch_list_total_us"] = round(tot, 1)
# 2. conv DRAM traffic per launch vs the library's algorithmic bytes
prof = json.load(open(f"{src}/step_profile.json")) if os.path.exists(f"{src}/step_profile.json") else []
if os.path.exists(f"{src}/block_dram.csv"):
    by_id = defaultdict(dict)
    for r in rows(f"{src}/block_dram.csv"):
        by_id[int(r["ID"])][r["Metric Name"]] = (float(r["Metric Value"].replace(",", "")), r["Metric Unit"])
    blks = [p for p in prof if p["kind"] == "block"]
    launches = []
    for i, (k, m) in enumerate(sorted(by_id.items())):
        rd = m["dram__bytes_read.sum"][0]
        wr = m["dram__bytes_write.sum"][0]
        t = m["gpu__time_duration.sum"]
        t_us = t[0] * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3}.get(t[1], 1.0)
        alg = blks[i]["bytes"] if i < len(blks) else None
        launches.append({"launch": i, "dram_bytes": rd + wr, "algorithmic_bytes": alg, "ncu_us": t_us,
                         "event_us": blks[i]["ms"] * 1e3 if i < len(blks) else None})
    tot_dram = sum(l["dram_bytes"] for l in launches)
    tot_alg = sum(l["algorithmic_bytes"] or 0 for l in launches)
    out["block_dram"] = {"launches": len(launches), "dram_bytes_per_launch": tot_dram / len(launches),
                         "algorithmic_bytes_per_launch": tot_alg / len(launches),
                         "dram_over_algorithmic": tot_dram / tot_alg if tot_alg else None,
                         "per_launch": launches}
    json.dump({"kernel": "k_block_fused", "dram_bytes_per_launch": tot_dram / len(launches),
               "algorithmic_bytes_per_launch": tot_alg / len(launches),
               "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over the {len(launches)} "
                         f"k_block_fused launches of one cfg2 step (profiles/{tag}_profile.json)"},
              open("profiles/block_traffic.json", "w"), indent=1)
if os.path.exists(f"{src}/conv_dram.csv"):
    by_id = defaultdict(dict)
    for r in rows(f"{src}/conv_dram.csv"):
        by_id[int(r["ID"])][r["Metric Name"]] = (float(r["Metric Value"].replace(",", "")), r["Metric Unit"])
    convs = [p for p in prof if p["kind"] == "conv"]
    launches = []
    for i, (k, m) in enumerate(sorted(by_id.items())):
        rd = m["dram__bytes_read.sum"][0]
        wr = m["dram__bytes_write.sum"][0]
        t = m["gpu__time_duration.sum"]
        t_us = t[0] * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3}.get(t[1], 1.0)
        alg = convs[i]["bytes"] if i < len(convs) else None
        launches.append({"launch": i, "dram_bytes": rd + wr, "algorithmic_bytes": alg, "ncu_us": t_us,
                         "event_us": convs[i]["ms"] * 1e3 if i < len(convs) else None})
    tot_dram = sum(l["dram_bytes"] for l in launches)
    tot_alg = sum(l["algorithmic_bytes"] or 0 for l in launches)
    out["conv_dram"] = {"launches": len(launches), "dram_bytes_per_launch": tot_dram / len(launches),
                        "algorithmic_bytes_per_launch": tot_alg / len(launches),
                        "dram_over_algorithmic": tot_dram / tot_alg if tot_alg else None,
                        "per_launch": launches}
    json.dump({"dram_bytes_per_launch": tot_dram / len(launches),
               "algorithmic_bytes_per_launch": tot_alg / len(launches),
               "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over the {len(launches)} conv "
                         f"launches of one cfg2 step (profiles/{tag}_profile.json)"},
              open("profiles/conv_traffic.json", "w"), indent=1)
if prof:
    agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for p in prof:
        a = agg[p["kind"]]
        a[0] += 1
        a[1] += p["ms"]
        a[2] += p["bytes"]
        a[3] += p["flops"]
    out["event_timed_step"] = {k: {"launches": v[0], "ms": round(v[1], 4),
                                   "GB_per_s": round(v[2] / v[1] / 1e6, 1) if v[1] else None,
                                   "TFLOP_per_s": round(v[3] / v[1] / 1e9, 1) if v[1] else None}
                               for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}
json.dump(out, open(f"profiles/{tag}_profile.json", "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "conv_dram"}, indent=1))
if "conv_dram" in out:
    c = out["conv_dram"]
    print("conv dram/launch %.3g MB, algorithmic %.3g MB, ratio %.2f" % (
        c["dram_bytes_per_launch"] / 1e6, c["algorithmic_bytes_per_launch"] / 1e6, c["dram_over_algorithmic"]))
