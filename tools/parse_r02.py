"""Round-2 evidence summaries: gpurun_out/ (tools/profile_r02.sh) -> profiles/r02_*.

  profiles/r02_launches_cfg{5,2,4}.json  per-kernel share of one chunk / step (ncu launch list:
                                          serialised, cold caches -> compare SHARES) + DRAM bytes
  profiles/r02_traffic.json              ncu DRAM read+write bytes per launch of the bench's
                                          dominant kernel class (bench.py roofline.traffic)
  profiles/r02_ncu_*.txt                 --set full summaries (tools/ncu_summary.py)
  profiles/r02_sanitizers.txt            racecheck / synccheck / memcheck verdict lines
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
os.makedirs("profiles", exist_ok=True)
UNIT = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def launches(path):
    lines = [l for l in open(path) if l.startswith('"')]
    per = defaultdict(dict)
    names = {}
    for r in csv.DictReader(lines):
        i = int(r["ID"])
        names[i] = r["Kernel Name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "") \
            .replace("dycl::", "").replace("unnamed>::", "")
        v = float(r["Metric Value"].replace(",", ""))
        u = r["Metric Unit"]
        if r["Metric Name"] == "gpu__time_duration.sum":
            per[i]["us"] = v * UNIT.get(u, 1.0)
        else:
            per[i][r["Metric Name"]] = v * BYTES.get(u, 1.0)
    out = []
    for i in sorted(per):
        d = per[i]
        out.append(dict(id=i, kernel=names[i], us=round(d.get("us", 0.0), 2),
                        dram_bytes=d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)))
    return out


def summarise(L):
    per = defaultdict(lambda: [0, 0.0, 0.0])
    for l in L:
        k = l["kernel"].split("<")[0]
        per[k][0] += 1
        per[k][1] += l["us"]
        per[k][2] += l["dram_bytes"]
    tot = sum(v[1] for v in per.values()) or 1.0
    return {k: {"launches": v[0], "us": round(v[1], 1), "share": round(v[1] / tot, 4),
                "dram_bytes_per_launch": v[2] / v[0], "dram_GBps": v[2] / (v[1] * 1e3) if v[1] else 0.0}
            for k, v in sorted(per.items(), key=lambda kv: -kv[1][1])}, tot


traffic = {}
for cfg, dom, kern in [(5, "conv", "k_conv_gemm"), (2, "block", "k_block_fused"), (4, "gemm", "k_gemm_tma")]:
    p = f"{src}/c{cfg}_launches.csv"
    if not os.path.exists(p):
        continue
    L = launches(p)
    summ, tot = summarise(L)
    json.dump({"source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                         f"--clock-control none, one {'2048-row chunk' if cfg == 5 else 'batch'} of config {cfg} "
                         f"run launch by launch (graph off); serialised + cold caches: compare shares",
               "total_us": round(tot, 1), "per_kernel": summ, "launches": L},
              open(f"profiles/r02_launches_cfg{cfg}.json", "w"), indent=1)
    if kern in summ and summ[kern]["dram_bytes_per_launch"] > 0:
        traffic[f"cfg{cfg}"] = {dom: {"kernel": kern, "dram_bytes_per_launch": summ[kern]["dram_bytes_per_launch"],
                                      "launches": summ[kern]["launches"]}}
    print(f"cfg{cfg}: total {tot:.0f} us;", ", ".join(f"{k} {v['share']:.2f}" for k, v in list(summ.items())[:6]))
if traffic:
    json.dump(traffic, open("profiles/r02_traffic.json", "w"), indent=1)
for rep, name in [("c5_conv_full", "r02_ncu_conv_gemm_cfg5.txt"), ("c2_block_full", "r02_ncu_block_fused_cfg2.txt")]:
    f = f"{src}/{rep}.ncu-rep"
    if os.path.exists(f):
        out = subprocess.run([sys.executable, "tools/ncu_summary.py", f, "15"], capture_output=True, text=True).stdout
        open(f"profiles/{name}", "w").write(out)
        print("wrote", name)
san = []
for tool in ["racecheck", "synccheck", "memcheck"]:
    for ext in ("log", "out"):
        f = f"{src}/{tool}_r02.{ext}"
        if os.path.exists(f):
            lines = open(f).read().strip().splitlines()
            san.append(f"== {tool} ({ext}) ==")
            san += [l for l in lines if "ERROR SUMMARY" in l or "passed" in l or "failed" in l or "Error" in l][-6:]
if san:
    open("profiles/r02_sanitizers.txt", "w").write("\n".join(san) + "\n")
    print("\n".join(san))
