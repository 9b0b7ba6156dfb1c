"""Summarise an ncu report: key SOL metrics + top source lines by stall samples."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
want = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issued Instructions", "Registers Per Thread",
        "Achieved Active Warps Per SM", "L1/TEX Hit Rate", "L2 Hit Rate", "Eligible Warps Per Scheduler",
        "No Eligible", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block"]
seen = set()
for r in rows[1:]:
    d = dict(zip(hdr, r))
    k = d.get("Metric Name")
    if k in want and (d.get("Kernel Name"), k) not in seen:
        seen.add((d.get("Kernel Name"), k))
        print(f"  {k:40s} {d.get('Metric Value'):>14s} {d.get('Metric Unit')}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) > 2:
    h = rr[0]
    for ki in range(2, len(rr)):
        kn = rr[ki][h.index("Kernel Name")] if "Kernel Name" in h else f"kernel {ki - 2}"
        print(f"  [launch {ki - 2}] {kn[:90]}")
        for name in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                     "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                     "sm__inst_executed_pipe_tensor.sum", "l1tex__t_bytes.sum", "lts__t_bytes.sum",
                     "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active"]:
            for i, col in enumerate(h):
                if col.startswith(name):
                    print(f"    {col:60s} {rr[ki][i]:>16s} {rr[1][i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
for hi, r in enumerate(rows):
    if "Warp Stall Sampling (All Samples)" in r:
        break
else:
    sys.exit(0)
hdr = rows[hi]
S = hdr.index("Warp Stall Sampling (All Samples)")
I = hdr.index("Instructions Executed")
lines = [r for r in rows[hi + 1:] if len(r) > S and r[0] != ""]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot = sum(f(r[S]) for r in lines) or 1
ti = sum(f(r[I]) for r in lines) or 1
print(f"  top source lines (stall samples {tot:.0f}, instructions {ti:.3g}):")
for r in sorted(lines, key=lambda r: -f(r[S]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(f"   L{r[0]:>4} {f(r[S]) / tot * 100:5.1f}% inst {f(r[I]) / ti * 100:5.1f}%  {r[1][:96]}")
