"""Summarise ncu captures into profiles/ (run here, on the CPU, from gpurun_out/ files).

usage: python tools/summarize_profile.py <launches.csv> <prof.ncu-rep> <bench.json> <out.md>
"""
import collections
import csv
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].replace("nsdf_b200::", "").replace("<unnamed>::", "")
        agg[name[:90]][0] += 1
        agg[name[:90]][1] += float(d["Metric Value"])
    return agg


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u, v = r[0], r[1], r[2]
    d = {h[i]: (v[i], u[i]) for i in range(len(h))}
    return d


def main():
    lp, rep, bj, out = sys.argv[1:5]
    agg = launches(lp)
    tot = sum(v[1] for v in agg.values())
    d = raw(rep)
    bench = json.loads(open(bj).read().strip().splitlines()[-1])
    lines = ["# Profile summary", "",
             f"Bench line (`python bench.py`, defaults): {bench['value']:.1f} {bench['unit']}, "
             f"{bench['ms_per_step']:.3f} ms/frame, e2e {bench['e2e']['value']:.1f} {bench['e2e']['unit']}, "
             f"roofline frac {bench['roofline']['frac']:.3f} ({bench['roofline']['achieved']:.1f} of "
             f"{bench['roofline']['peak']:.1f} TFLOP/s), CPU reference {bench['cpu_baseline']['value']:.3f} "
             f"{bench['cpu_baseline']['unit']} on {bench['cpu_baseline']['cores']} cores, clocks {bench['clocks']}", "",
             "## Launch list (ncu `gpu__time_duration.sum`, cold-cache, serialised: compare shares)", "",
             "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {v[0]} | {v[1] / 1e3:.1f} | {100 * v[1] / tot:.1f}% |")
    lines += ["", f"## Top kernel: `ncu --set full` of one launch ({rep.split('/')[-1]})", "",
              "| metric | value |", "|---|---|"]
    for m in METRICS:
        if m in d:
            lines.append(f"| {m} | {d[m][0]} {d[m][1]} |")
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): v[0] for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    top = sorted(((k, int(float(v.replace(",", "")))) for k, v in stalls.items() if v), key=lambda x: -x[1])[:8]
    lines += ["", "Top warp-stall samples: " + ", ".join(f"{k} {v}" for k, v in top), ""]
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
