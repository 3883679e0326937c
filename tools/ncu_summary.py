"""Summarise a gpurun's ncu output into profiles/ (tracked).

    python tools/ncu_summary.py TAG [--launches gpurun_out/launches_TAG.csv]
                                    [--rep gpurun_out/prof_sweep_TAG.ncu-rep] [--out profiles/]

Writes profiles/<TAG>_launches.md (per-kernel share of the step from the
`--metrics gpu__time_duration.sum` pass) and profiles/<TAG>_sweep_ncu.md (the
`--set full` capture of the dominant kernel: duration, issue/tensor/DRAM
figures, registers, and the per-instruction hot spots of the source page).
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _kernel_short(name: str) -> str:
    name = name.replace("<unnamed>::", "").replace("void ", "")
    if "(" in name:
        name = name[:name.index("(")]
    return name.strip()


def launches(path: str) -> str:
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg: "OrderedDict[str, list]" = OrderedDict()
    unit = None
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        unit = r[ui]
        agg.setdefault(_kernel_short(r[ki]), []).append(float(r[vi].replace(",", "")))
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3}.get(unit, 1.0)
    ours = {k: v for k, v in agg.items() if not k.startswith("at::")}
    per_step = {k: sum(v) / len(v) * scale for k, v in ours.items()}
    total = sum(per_step.values())
    out = ["| kernel | launches | mean us/launch | share of our kernels' time per step |",
           "|---|---|---|---|"]
    for k, v in sorted(per_step.items(), key=lambda kv: -kv[1]):
        out.append(f"| `{k}` | {len(ours[k])} | {v:.2f} | {v / total:.1%} |")
    other = {k: v for k, v in agg.items() if k.startswith("at::")}
    if other:
        out.append("")
        out.append("torch launches in the same process (L2-flush memsets, buffer zeroing; "
                   "outside the timed step events): " +
                   ", ".join(f"`{k[:50]}` x{len(v)}" for k, v in other.items()))
    return "\n".join(out)


def _ncu(rep: str, *args) -> str:
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


RAW_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy"),
    ("sm__inst_executed.sum.pct_of_peak_sustained_elapsed", "SM instruction throughput (of peak, elapsed)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active"),
    ("sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active", "tensor (hmma subpipe) inst"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 traffic"),
]


def full(rep: str, top: int = 40) -> str:
    raw = list(csv.reader(io.StringIO(_ncu(rep, "--page", "raw", "--csv"))))
    out = []
    if len(raw) >= 3:
        h, u = raw[0], raw[1]
        for row in raw[2:]:
            name = row[h.index("Kernel Name")] if "Kernel Name" in h else "?"
            out.append(f"### `{_kernel_short(name)}`\n")
            out.append("| metric | value |\n|---|---|")
            for key, label in RAW_METRICS:
                if key in h:
                    i = h.index(key)
                    out.append(f"| {label} (`{key}`) | {row[i]} {u[i]} |")
            out.append("")
    src = list(csv.reader(io.StringIO(_ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    # one section per profiled kernel: a "Kernel Name" row, a header row, the body
    sections, cur = [], None
    for row in src:
        if row and row[0] == "Kernel Name":
            cur = {"name": row[1] if len(row) > 1 else "?", "rows": []}
            sections.append(cur)
        elif cur is not None:
            cur["rows"].append(row)
    for sec in sections:
        if len(sec["rows"]) < 2:
            continue
        h = sec["rows"][0]
        ia, ie = h.index("Source"), h.index("Instructions Executed")
        iss = h.index("Warp Stall Sampling (All Samples)")
        body = [r for r in sec["rows"][1:] if len(r) == len(h)]
        tot_e = sum(int(r[ie]) for r in body)
        tot_s = sum(int(r[iss]) for r in body) or 1
        out.append(f"Source page of `{_kernel_short(sec['name'])}`: {tot_e} warp instructions "
                   f"executed, {tot_s} stall samples.\n")
        out.append(f"Top {top} SASS lines by stall samples:\n")
        out.append("| addr | executed | stall samples | SASS |\n|---|---|---|---|")
        for r in sorted(body, key=lambda r: -int(r[iss]))[:top]:
            out.append(f"| {r[0][-5:]} | {r[ie]} | {r[iss]} | `{r[ia].strip()}` |")
        out.append("")
    return "\n".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles"))
    ap.add_argument("--note", default="")
    ap.add_argument("--traffic-key", default=None,
                    help="WORKLOAD/KERNEL: record the first captured kernel's DRAM bytes "
                         "(read + write) in profiles/traffic.json for bench.py's roofline")
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    lp = a.launches or os.path.join(ROOT, "gpurun_out", f"launches_{a.tag}.csv")
    rp = a.rep or os.path.join(ROOT, "gpurun_out", f"prof_sweep_{a.tag}.ncu-rep")
    if os.path.exists(lp):
        with open(os.path.join(a.out, f"{a.tag}_launches.md"), "w") as fh:
            fh.write(f"# {a.tag}: launch list (`ncu --metrics gpu__time_duration.sum "
                     f"--clock-control none`)\n\n{a.note}\n\n")
            fh.write("Cold-cache, serialised per-launch times: compare shares, not absolutes.\n\n")
            fh.write(launches(lp) + "\n")
    if os.path.exists(rp):
        with open(os.path.join(a.out, f"{a.tag}_sweep_ncu.md"), "w") as fh:
            fh.write(f"# {a.tag}: `ncu --set full --clock-control none --import-source on` "
                     f"of the dominant kernel\n\n{a.note}\n\n")
            fh.write(full(rp) + "\n")
        if a.traffic_key:
            raw = list(csv.reader(io.StringIO(_ncu(rp, "--page", "raw", "--csv"))))
            h, u, row = raw[0], raw[1], raw[2]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tot = sum(float(row[h.index(k)]) * scale.get(u[h.index(k)], 1)
                      for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            path = os.path.join(a.out, "traffic.json")
            d = json.load(open(path)) if os.path.exists(path) else {}
            d[a.traffic_key] = tot
            with open(path, "w") as fh:
                json.dump(d, fh, indent=1, sort_keys=True)
            # warp instructions executed by the captured launch (issue roofline)
            inst = float(row[h.index("smsp__inst_executed.sum")]) if "smsp__inst_executed.sum" in h else None
            if inst:
                path = os.path.join(a.out, "issue.json")
                d = json.load(open(path)) if os.path.exists(path) else {}
                d[a.traffic_key] = inst
                with open(path, "w") as fh:
                    json.dump(d, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
