"""Summarise ncu captures into profiles/ (run here, on the CPU, from gpurun_out/ files).

usage: python tools/summarize_profile.py <launches.csv> <full.ncu-rep> <bench.json> <out.md> [traffic.json]

<launches.csv>  `ncu --metrics gpu__time_duration.sum --clock-control none --csv` launch list of a
                bench run (cold-cache, serialised per-launch times: compare shares, not absolutes)
<full.ncu-rep>  `ncu --set full` capture of the tcgen05 kernels of one frame (one column each)
<bench.json>    the bench line of the same code
[traffic.json]  written: DRAM bytes per launch of each captured kernel (bench.py reads it for
                roofline.traffic)
"""
import collections
import csv
import json
import re
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads per warp instr (of 32)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "SMEM wavefronts %"),
    ("lts__t_sectors.avg.pct_of_peak_sustained_elapsed", "L2 sectors %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
]
UNIT_BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def short(name):
    m = re.search(r"tc_mlp_kernel<[^>]*>", name.replace("(int)", "").replace("(bool)", ""))
    if m:
        return m.group(0)
    name = re.sub(r"(nsdf_b200::|<?unnamed>::|void )", "", name)
    return name.split("(")[0][:60]


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
        name = short(d["Kernel Name"])
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"].replace(",", ""))
    return agg


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u = r[0], r[1]
    return [{h[i]: (v[i], u[i]) for i in range(len(h))} for v in r[2:]]


def main():
    lp, rep, bj, out = sys.argv[1:5]
    traffic_out = sys.argv[5] if len(sys.argv) > 5 else None
    agg = launches(lp)
    tot = sum(v[1] for v in agg.values())
    kern = raw(rep)
    bench = json.loads(open(bj).read().strip().splitlines()[-1])
    rf = bench["roofline"]
    lines = ["# Profile summary", "",
             f"Bench line (`python bench.py`, defaults): {bench['value']:.1f} {bench['unit']}, "
             f"{bench['ms_per_step']:.3f} ms/frame ({bench['fps']:.0f} fps), frames in flight "
             f"{bench['config'].get('frames_in_flight', 1)}; e2e {bench['e2e']['value']:.1f} {bench['e2e']['unit']}; "
             f"roofline frac {rf['frac']:.3f} ({rf['achieved']:.1f} of {rf['peak']:.1f} TFLOP/s, algorithmic); "
             f"MUFU activation frac {rf['activation_bound']['frac']:.3f}; CPU reference "
             f"{bench['cpu_baseline']['value']:.3f} {bench['cpu_baseline']['unit']} on {bench['cpu_baseline']['cores']} "
             f"cores; clocks {bench['clocks']}", "",
             "## Launch list (ncu `gpu__time_duration.sum`, cold-cache, serialised: compare shares)", "",
             "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {v[0]} | {v[1] / 1e3:.1f} | {100 * v[1] / tot:.1f}% |")
    names = [short(k["Kernel Name"][0]) for k in kern]
    lines += ["", f"## `ncu --set full` of one frame's tcgen05 kernels ({rep.split('/')[-1]})", "",
              "| metric | " + " | ".join(f"`{n}`" for n in names) + " |",
              "|---|" + "---|" * len(names)]
    for m, label in METRICS:
        vals = []
        for k in kern:
            v, u = k.get(m, ("-", ""))
            vals.append(f"{v} {u}".strip())
        lines.append(f"| {label} | " + " | ".join(vals) + " |")
    lines += ["", "Top warp-stall samples per kernel:", ""]
    traffic = {}
    for n, k in zip(names, kern):
        stalls = {key.replace("smsp__pcsamp_warps_issue_stalled_", ""): v[0] for key, v in k.items()
                  if key.startswith("smsp__pcsamp_warps_issue_stalled_") and not key.endswith("not_issued")}
        top = sorted(((s, int(float(v.replace(",", "")))) for s, v in stalls.items() if v and v != "n/a"),
                     key=lambda x: -x[1])[:8]
        tot_s = sum(v for _, v in top) or 1
        lines.append(f"- `{n}`: " + ", ".join(f"{s} {100 * v / tot_s:.0f}%" for s, v in top))
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v, u = k.get(m, ("0", "byte"))
            b += float(v.replace(",", "")) * UNIT_BYTES.get(u, 1)
        traffic[n] = b
    lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    if traffic_out:
        json.dump({"source": rep.split("/")[-1], "dram_bytes_per_launch": traffic}, open(traffic_out, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
