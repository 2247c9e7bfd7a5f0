"""Summarise ncu captures of the stitched kernels into profiles/.

    python profiles/ncu_summary.py <full.ncu-rep> [launches.csv] --tag r01

Writes profiles/<tag>_kernels.md (per-kernel DRAM bytes, DRAM/SM throughput,
occupancy, registers, top warp stalls from the `--set full` capture),
profiles/<tag>_launches.md (per-kernel share of the launch list from the
`--metrics gpu__time_duration.sum` pass of bench.py) and merges the per-launch
DRAM traffic into profiles/traffic.json, which bench.py reports as
roofline.traffic for the dominant kernel.
"""

from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))

METRICS = {
    "dur_us": "gpu__time_duration.sum",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "inst": "smsp__inst_executed.sum",
    "l2_hit": "lts__t_sector_hit_rate.pct",
    "bank_conflicts_ld": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "bank_conflicts_st": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "smem_wavefronts_ld": "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "smem_wavefronts_st": "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
    "occ_theory": "sm__maximum_warps_per_active_cycle_pct",
    # L2 write sectors from the SMs: the kernel's stores even when the output
    # is still in L2 (not yet written back to DRAM) when the capture ends
    "l2_wr_sectors": "lts__t_sectors_srcunit_tex_op_write.sum",
}

UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1, "ms": 1e3, "ns": 1e-3, "s": 1e6}


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k, m in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[k] = v * UNIT_SCALE.get(units[i], 1)
        stalls = {}
        for i, h in enumerate(hdr):
            pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
            if h.startswith(pre) and h.endswith(suf):
                try:
                    stalls[h[len(pre):-len(suf)]] = float(r[i])
                except ValueError:
                    pass
        d["stalls"] = sorted(stalls.items(), key=lambda kv: -kv[1])[:4]
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("launches", nargs="?")
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--algo", default=None, help="json {kernel: algorithmic bytes per launch}")
    ap.add_argument("--config", required=True, help="workload name (keys of traffic.json are <config>/<kernel>)")
    args = ap.parse_args()
    algo = json.load(open(args.algo)) if args.algo else {}
    rows = raw_rows(args.rep)
    lines = [f"# ncu --set full summary ({args.tag})", "",
             f"source: `{os.path.basename(args.rep)}` (ncu --set full --clock-control none, cold cache, "
             "serialised replay; compare shares, not absolutes)", "",
             "`L2 wr MB` = lts__t_sectors_srcunit_tex_op_write × 32 B: the kernel's stores as L2 sees them, "
             "so `(DRAM rd + L2 wr) / algo` confirms full writes even when the output is still in L2 "
             "(not yet in DRAM) when the capture ends.", "",
             "| kernel | dur us | DRAM rd MB | DRAM wr MB | L2 wr MB | DRAM GB/s | traffic/algo | (DRAM rd + L2 wr)/algo | DRAM % | SM % | occupancy achieved / theoretical % | smem bank conflicts ld / st (wavefronts) | regs | grid | top stalls |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    traffic_path = os.path.join(HERE, "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for d in rows:
        t = d.get("dram_rd", 0) + d.get("dram_wr", 0)
        a = algo.get(d["kernel"])
        ratio = f"{t / a:.3f}" if a else "-"
        l2w = d.get("l2_wr_sectors", 0) * 32
        ratio2 = f"{(d.get('dram_rd', 0) + l2w) / a:.3f}" if a else "-"
        gbs = t / (d["dur_us"] * 1e3) if d.get("dur_us") else 0.0
        bc = (f"{int(d.get('bank_conflicts_ld', 0))} / {int(d.get('bank_conflicts_st', 0))} "
              f"({int(d.get('smem_wavefronts_ld', 0))} / {int(d.get('smem_wavefronts_st', 0))})")
        lines.append(f"| {d['kernel']} | {d.get('dur_us', 0):.1f} | {d.get('dram_rd', 0) / 1e6:.1f} | "
                     f"{d.get('dram_wr', 0) / 1e6:.1f} | {l2w / 1e6:.1f} | {gbs:.0f} | {ratio} | {ratio2} | "
                     f"{d.get('dram_pct', 0):.1f} | "
                     f"{d.get('sm_pct', 0):.1f} | {d.get('warps_active_pct', 0):.1f} / {d.get('occ_theory', 0):.1f} | {bc} | "
                     f"{int(d.get('regs', 0))} | {int(d.get('grid', 0))} | "
                     + ", ".join(f"{k} {v:.1f}" for k, v in d["stalls"]) + " |")
        traffic[f"{args.config}/{d['kernel']}"] = t
    with open(os.path.join(HERE, f"{args.tag}_kernels.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(traffic_path, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)
    if args.launches:
        per = collections.defaultdict(list)
        with open(args.launches) as f:
            text = [l for l in f if not l.startswith("==")]
        rd = csv.DictReader(io.StringIO("".join(text)))
        for r in rd:
            if r.get("Metric Name") == "gpu__time_duration.sum":
                v = float(r["Metric Value"].replace(",", ""))
                scale = UNIT_SCALE.get(r.get("Metric Unit", "ns"), 1e-3)
                per[r["Kernel Name"]].append(v * scale)
        total = sum(sum(v) for v in per.values())
        out = [f"# launch list ({args.tag})", "",
               f"source: `{os.path.basename(args.launches)}` (ncu --metrics gpu__time_duration.sum "
               "--clock-control none over bench.py)", "",
               "| kernel | launches | mean us | share of device time |", "|---|---|---|---|"]
        for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            name = k if len(k) < 60 else k[:57] + "..."
            out.append(f"| {name} | {len(v)} | {sum(v) / len(v):.1f} | {100 * sum(v) / total:.1f}% |")
        with open(os.path.join(HERE, f"{args.tag}_launches.md"), "w") as f:
            f.write("\n".join(out) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
