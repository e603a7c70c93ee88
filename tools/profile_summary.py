"""Summarise ncu output into profiles/ (committed evidence).

    python tools/profile_summary.py launches gpurun_out/launches.csv > profiles/rNN_launches.md
    python tools/profile_summary.py full gpurun_out/prof.ncu-rep [label] > profiles/rNN_<kernel>.md

`full` also prints the per-launch DRAM traffic used as roofline.traffic.
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(list)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                agg[d["Kernel Name"]].append(float(d["Metric Value"]))
    tot = sum(sum(v) for v in agg.values())
    print(f"# ncu launch list: {path}\n")
    print("cold-cache, serialised per-launch times (`--metrics gpu__time_duration.sum "
          "--clock-control none`): compare shares, not absolutes.\n")
    print("| kernel | launches | total ms | mean ms | share |\n|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"| `{k[:90]}` | {len(v)} | {sum(v) / 1e6:.3f} | {sum(v) / len(v) / 1e6:.3f} | "
              f"{sum(v) / tot:.3f} |")


def full(path, label=""):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full: {label or path}\n")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"## `{d.get('Kernel Name', '?')[:100]}`\n")
        print("| metric | value | unit |\n|---|---|---|")
        for k in KEYS:
            if k in d:
                print(f"| {k} | {d[k]} | {u.get(k, '')} |")
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
        try:
            rb = float(d["dram__bytes_read.sum"]) * scale.get(u["dram__bytes_read.sum"], 1.0)
            wb = float(d["dram__bytes_write.sum"]) * scale.get(u["dram__bytes_write.sum"], 1.0)
            print(f"\nDRAM traffic per launch: {rb + wb:.4g} bytes (read {rb:.4g}, write {wb:.4g})\n")
        except (KeyError, ValueError):
            pass
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    if src:
        print("## hottest source lines (warp-stall samples / executed instructions)\n\n```")
        tmp = "/tmp/_src.csv"
        open(tmp, "w").write(src)
        out = subprocess.run([sys.executable, __file__.replace("profile_summary.py", "ncu_lines.py"),
                              tmp, "25"], capture_output=True, text=True).stdout
        print(out.rstrip())
        print("```")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
