"""Summarise ncu captures into profiles/ (tracked).

    python tools/ncu_summary.py <tag> gpurun_out/prof_aa.ncu-rep [gpurun_out/launches.csv]

Writes profiles/<tag>_kernels.md (per-kernel DRAM bytes, duration,
registers, occupancy, throughput %, algorithmic bytes and the ratio) and
updates profiles/latest_traffic.json, which bench.py reports as
roofline.traffic.
"""

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__maximum_warps_per_active_cycle_pct",
    "lts__t_sector_hit_rate.pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "launch__grid_size",
    "launch__block_size",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
         "nsecond": 1e-9, "second": 1.0}


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    return rows[0], rows[1], rows[2:]


def to_si(val, unit):
    try:
        v = float(val.replace(",", ""))
    except ValueError:
        return val
    return v * SCALE.get(unit, 1.0)


def algorithmic_bytes(name, n_cells):
    q = 27 if "D3Q27" in name else (9 if "D2Q9" in name else 19)
    if "aa_odd" in name:
        return 2 * q * 8 * n_cells
    if "aa_even" in name or "pull" in name or "index_sweep" in name:
        return (2 * q * 8 + (q - 1) * 4) * n_cells
    if "k_group_hot<" in name or "k_group<" in name:
        # block-group sweeps over every engine of the group: template
        # arguments <lattice, model, KIND[, CAP]>, KIND 2 = cell-local
        fn = "k_group_hot<" if "k_group_hot<" in name else "k_group<"
        kind = int(name.split(fn, 1)[1].split(">")[0].split(",")[2])
        return (2 * q * 8 + (0 if kind == 2 else (q - 1) * 4)) * n_cells
    return None


def main():
    tag, rep = sys.argv[1], sys.argv[2]
    n_cells = int(os.environ.get("N_FLUID", "40267378"))
    h, units, rows = raw_rows(rep)
    ki = h.index("Kernel Name")
    lines = [f"# ncu summary {tag}", "", f"source: `{os.path.basename(rep)}` (ncu --set full, "
             f"--clock-control none); n_fluid per launch = {n_cells}", "",
             "| kernel | ms | DRAM read GB | DRAM write GB | traffic/algorithmic | DRAM % peak | regs | "
             "occupancy % (active/max) | L2 hit % | fp64 pipe % |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for r in rows:
        m = {k: to_si(r[h.index(k)], units[h.index(k)]) for k in METRICS if k in h}
        name = r[ki]
        short = name.split("(")[0].replace("void ", "").replace("slbm::", "").replace("<unnamed>::", "")
        tot = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        alg = algorithmic_bytes(name, n_cells)
        ratio = f"{tot / alg:.3f}" if alg else "-"
        lines.append(
            f"| `{short}` | {m['gpu__time_duration.sum'] * 1e3:.3f} | {m['dram__bytes_read.sum'] / 1e9:.3f} | "
            f"{m['dram__bytes_write.sum'] / 1e9:.3f} | {ratio} | "
            f"{m['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']:.1f} | "
            f"{int(m['launch__registers_per_thread'])} | "
            f"{m['sm__warps_active.avg.pct_of_peak_sustained_active']:.1f}/"
            f"{m['sm__maximum_warps_per_active_cycle_pct']:.1f} | {m['lts__t_sector_hit_rate.pct']:.1f} | "
            f"{m['sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active']:.1f} |")
        idx_sweep = "aa_even" in name or "index_sweep" in name
        key = "k_aa_even" if idx_sweep else ("k_aa_odd" if "aa_odd" in name else short)
        traffic.setdefault(key, []).append(tot)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{tag}_kernels.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    latest = {f"{k}_dram_bytes_per_launch": sum(v) / len(v) for k, v in traffic.items()}
    latest["source"] = f"profiles/{tag}_kernels.md"
    if os.environ.get("NO_TRAFFIC") != "1":  # other workloads must not feed the bench line
        with open(os.path.join(ROOT, "profiles", "latest_traffic.json"), "w") as fh:
            json.dump(latest, fh, indent=1)
    print("\n".join(lines))
    if len(sys.argv) > 3:
        summarize_launches(tag, sys.argv[3])


def summarize_launches(tag, path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = {}
    order = []
    for r in rows[hdr + 1:]:
        name = r[ki].split("(")[0].replace("void ", "").replace("slbm::", "").replace("<unnamed>::", "")
        t = to_si(r[vi], r[ui])
        if name not in agg:
            order.append(name)
            agg[name] = []
        agg[name].append(t)
    total = sum(sum(v) for v in agg.values())
    lines = [f"# launch list {tag}", "", "ncu --metrics gpu__time_duration.sum --clock-control none "
             "(cold-cache, serialised; compare shares)", "",
             "| kernel | launches | mean ms | total ms | share % |", "|---|---|---|---|---|"]
    for name in order:
        v = agg[name]
        lines.append(f"| `{name}` | {len(v)} | {sum(v) / len(v) * 1e3:.4f} | {sum(v) * 1e3:.3f} | "
                     f"{100 * sum(v) / total:.1f} |")
    with open(os.path.join(ROOT, "profiles", f"{tag}_launches.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
