"""Summarise ncu reports / launch lists into profiles/ (markdown + json).

    python scripts/ncu_summary.py report gpurun_out/fwd_h33_r01.ncu-rep profiles/r01_fwd_h33.md
    python scripts/ncu_summary.py launches gpurun_out/launches_fwd_r01.csv profiles/r01_launches_fwd.md
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active (% of peak)"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe (MUFU) %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes_read.sum.per_second", "DRAM read BW"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
]
STALLS = ["long_scoreboard", "barrier", "wait", "branch_resolving", "short_scoreboard", "math_pipe_throttle",
          "no_instruction", "not_selected", "selected", "mio_throttle", "dispatch_stall"]

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def to_bytes(val, unit):
    return float(val.replace(",", "")) * UNIT.get(unit, 1)


def report(rep, out_md, traffic_json=None, config=None):
    hdr, units, rows = raw_rows(rep)
    idx = {k: i for i, k in enumerate(hdr)}
    lines = [f"# ncu summary: `{rep.split('/')[-1]}`", "",
             "Captured with `ncu --set full --clock-control none --import-source on` on one B200 "
             "(per-launch, cold-cache, serialized; compare shares, not absolute time).", ""]
    traffic = {}
    for r in rows:
        name = r[idx["Kernel Name"]]
        lines += [f"## {name[:120]}", "", "| metric | value |", "|---|---|"]
        for key, label in KEYS:
            if key in idx:
                lines.append(f"| {label} (`{key}`) | {r[idx[key]]} {units[idx[key]]} |")
        stall = {}
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in idx:
                stall[s] = float(r[idx[k]].replace(",", ""))
        if stall:
            top = sorted(stall.items(), key=lambda kv: -kv[1])[:6]
            lines.append("| top stall reasons (warps per issue) | " + ", ".join(f"{k} {v:.2f}" for k, v in top) + " |")
        rb = to_bytes(r[idx["dram__bytes_read.sum"]], units[idx["dram__bytes_read.sum"]])
        wb = to_bytes(r[idx["dram__bytes_write.sum"]], units[idx["dram__bytes_write.sum"]])
        lines.append(f"| DRAM traffic per launch (read + write) | {rb + wb:.4g} B |")
        lines.append("")
        traffic[name.split("(")[0].strip()] = rb + wb
    with open(out_md, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    if traffic_json and config:
        try:
            with open(traffic_json) as fh:
                data = json.load(fh)
        except Exception:
            data = {}
        fwd = [v for k, v in traffic.items() if "attn_fwd" in k]
        if fwd:
            data[config] = fwd[0]
        with open(traffic_json, "w") as fh:
            json.dump(data, fh, indent=1)


def launches(csv_path, out_md):
    rows = list(csv.reader(open(csv_path)))
    hdr = None
    recs = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                recs.append((d["Kernel Name"], float(d["Metric Value"].replace(",", "")), d["Metric Unit"]))
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}
    total = sum(v * scale.get(u, 1e-6) for _, v, u in recs)
    ours = [(n, v * scale.get(u, 1e-6)) for n, v, u in recs if "radial" in n or "list_" in n or "scan_rows" in n
            or "bwd_prep" in n]
    lines = [f"# launch list: `{csv_path.split('/')[-1]}`", "",
             "`ncu --metrics gpu__time_duration.sum --clock-control none` (serialized, cold-cache).", "",
             "| # | kernel | ms | share of all launches |", "|---|---|---|---|"]
    for i, (n, v, u) in enumerate(recs):
        ms = v * scale.get(u, 1e-6)
        lines.append(f"| {i} | `{n[:90]}` | {ms:.4f} | {100 * ms / total:.1f}% |")
    lines += ["", f"Total {total:.3f} ms over {len(recs)} launches; radial kernels {sum(m for _, m in ours):.3f} ms."]
    with open(out_md, "w") as fh:
        fh.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "report":
        report(sys.argv[2], sys.argv[3], *(sys.argv[4:6] if len(sys.argv) >= 6 else (None, None)))
    else:
        launches(sys.argv[2], sys.argv[3])
