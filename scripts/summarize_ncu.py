#!/usr/bin/env python
"""Summarise ncu artefacts into profiles/ (run here, after gpurun brings
the raw files back into gpurun_out/).

  python scripts/summarize_ncu.py launches <launches.csv> <out.md>
  python scripts/summarize_ncu.py full <report.ncu-rep> <out.md> [--traffic-key KEY]
"""

import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

UNIT = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0,
        "msecond": 1.0, "s": 1e3, "second": 1e3}


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = collections.defaultdict(lambda: [0, 0.0])
    order = []
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]]
        short = name.split("(")[0][:80]
        ms = float(r[ix["Metric Value"]].replace(",", "")) * UNIT[r[ix["Metric Unit"]]]
        agg[short][0] += 1
        agg[short][1] += ms
        order.append((short, ms))
    total = sum(v[1] for v in agg.values())
    with open(out, "w") as fh:
        fh.write(f"# ncu launch list: `{os.path.basename(path)}`\n\n")
        fh.write("Per-launch `gpu__time_duration.sum`, `--clock-control none`. The times are "
                 "serialised and cold-cache, so compare shares, not absolute times.\n\n")
        fh.write("| kernel | launches | total ms | share | mean ms |\n|---|---|---|---|---|\n")
        for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
            fh.write(f"| `{k}` | {n} | {ms:.2f} | {ms / total * 100:.1f}% | {ms / n:.3f} |\n")
        fh.write("\nIndividual walk-kernel launches (ms): ")
        fh.write(", ".join(f"{ms:.1f}" for k, ms in order if "walk_kernel" in k))
        fh.write("\n")
    print(open(out).read())


METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard", None),
    ("smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.ratio",
     "global-load sector efficiency: bytes used per 32-B sector"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "global-load L1 sectors"),
    ("memory_l2_theoretical_sectors_global", "L2 sectors requested by global accesses"),
    ("memory_l2_theoretical_sectors_global_ideal", "  ... ideal (fully coalesced)"),
    ("lts__t_sectors.sum", "L2 sectors (all)"),
    ("lts__t_sectors.sum.pct_of_peak_sustained_elapsed", "L2 sector throughput % of peak"),
    ("smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio", None),
]


def full(rep, out, traffic_key=None, alg_bytes=None, queries=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    with open(out, "w") as fh:
        fh.write(f"# ncu --set full: `{os.path.basename(rep)}`\n\n")
        for r in rows[2:]:
            d = dict(zip(hdr, r))
            u = dict(zip(hdr, units))
            fh.write(f"## `{d.get('Kernel Name', '?')[:100]}`\n\n| metric | value |\n|---|---|\n")
            for key, label in METRICS:
                if key in d and label:
                    fh.write(f"| {label} (`{key}`) | {d[key]} {u.get(key, '')} |\n")
            stalls = sorted(((k, d[k]) for k in d if k.startswith(
                "smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")),
                key=lambda kv: -float(kv[1] or 0))[:8]
            if stalls:
                fh.write("\nTop stall reasons, in warps per issue-active cycle:\n\n")
                for k, v in stalls:
                    fh.write(f"- `{k.replace('smsp__average_warps_issue_stalled_', '')}`: {v}\n")
            rd = float(d.get("dram__bytes_read.sum", "0").replace(",", "") or 0)
            wr = float(d.get("dram__bytes_write.sum", "0").replace(",", "") or 0)
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
            tb = rd * scale.get(u.get("dram__bytes_read.sum"), 1) + \
                wr * scale.get(u.get("dram__bytes_write.sum"), 1)
            fh.write(f"\nDRAM traffic per launch: {tb:.4g} bytes\n\n")
            if alg_bytes:
                fh.write(f"Algorithmic bytes of this launch: {alg_bytes:.4g} "
                         f"(DRAM traffic / algorithmic = {tb / alg_bytes:.3f})\n\n")
            if traffic_key:
                p = os.path.join(ROOT, "profiles", "walk_traffic.json")
                cur = json.load(open(p)) if os.path.exists(p) else {}
                def num(key):
                    try:
                        return float(d.get(key, "").replace(",", ""))
                    except ValueError:
                        return None
                cur[traffic_key] = {"dram_bytes": tb, "alg_bytes": alg_bytes, "queries": queries,
                                    "report": os.path.basename(rep),
                                    "kernel_ms": num("gpu__time_duration.sum"),
                                    "l2_sectors": num("lts__t_sectors.sum"),
                                    "l2_sector_pct_of_peak": num(
                                        "lts__t_sectors.sum.pct_of_peak_sustained_elapsed"),
                                    "sector_bytes_used": num(
                                        "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.ratio"),
                                    "issue_pct": num(
                                        "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                                    "warp_inst": num("smsp__inst_executed.sum")}
                json.dump(cur, open(p, "w"), indent=1)
    print(open(out).read())


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    if mode == "launches":
        launches(src, dst)
    else:
        def opt(name, conv=str):
            return conv(sys.argv[sys.argv.index(name) + 1]) if name in sys.argv else None
        full(src, dst, opt("--traffic-key"), opt("--alg-bytes", float), opt("--queries", int))
