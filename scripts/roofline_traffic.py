"""Builds profiles/roofline_traffic.json (read by bench.py's roofline report) and a text summary
from the ncu --set full raw exports of scripts/r02_final.sh (gpurun_out/raw_<name>.csv):

  python scripts/roofline_traffic.py gpurun_out profiles/r02

Per capture: DRAM bytes read + written (dram__bytes_read.sum + dram__bytes_write.sum), warp
instructions (smsp__inst_executed.sum), duration, IPC, issue-slot use, achieved occupancy, L2 hit
rate, L2 atomic / reduction sectors. For count_smem_kernel (8 launches = the two tiers of 4 calls)
the timed step is the last two launches; count_ref_kernel captures hold every launch of one call (tier 1,
tier 2, hash-class passes).
"""
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth.configs import CONFIGS  # noqa: E402

METRICS = {
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "inst": "smsp__inst_executed.sum",
    "ms": "gpu__time_duration.sum",
    "ipc": "sm__inst_executed.avg.per_cycle_active",
    "issue": "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
    "occ": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l2hit": "lts__t_sector_hit_rate.pct",
    "atom": "lts__t_sectors_srcunit_tex_op_atom.sum",
    "red": "lts__t_sectors_srcunit_tex_op_red.sum",
    "dram_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
}
UNIT = {"dram_read": 1, "dram_write": 1}


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        d = {}
        for key, m in METRICS.items():
            if m not in hdr:
                continue
            i = hdr.index(m)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i].strip().lower()
            scale = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12,
                     "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(u, 1.0)
            d[key] = v * scale
        d["kernel"] = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""
        out.append(d)
    return out


SPECS = {  # capture name: (config, kernel label, launches per timed step)
    "c1_smem": ("C1", "count_smem_kernel", 2),
    "c1_supermer": ("C1", "supermer_kernel", 1),
    "c1_part": ("C1", "partition64_kernel", 2),
    "c1_regroup": ("C1", "regroup_counted_kernel", 1),
    "c1_ghist": ("C1", "group_hist_kernel", 1),
    "c4_ref": ("C4", "count_ref_kernel", 1),  # the tier-1 launch (~90 % of the reference-table time)
    "c4_supermer": ("C4", "supermer_kernel", 1),
}


def main():
    src, prefix = sys.argv[1], sys.argv[2]
    table, lines = [], []
    for name, (cfg, label, per_step) in SPECS.items():
        p = os.path.join(src, f"raw_{name}.csv")
        if not os.path.exists(p):
            continue
        launches = load(p)
        if not launches:
            continue
        if per_step is None:
            per_step = len(launches)
        step = launches[-per_step:]
        tot = lambda k: sum(x.get(k, 0.0) for x in step)  # noqa: E731
        dram = tot("dram_read") + tot("dram_write")
        c = CONFIGS[cfg]
        e = {"config": cfg, "k": c.k, "m": c.m, "kernel": label,
             "source": f"{prefix}_ncu_{name}.txt (ncu --set full --clock-control none, "
                       + (f"the timed step's {per_step} launch(es)" if name != "c4_ref" else
                          "the tier-1 launch of the first call (one of the step's reference-table launches)")
                       + f" of bench.py --config {cfg})",
             "launches": per_step, "ms_per_step": tot("ms"),
             "dram_bytes_per_launch": dram / per_step, "dram_bytes_per_step": dram,
             "warp_inst_per_step": tot("inst"),
             "ipc": sum(x.get("ipc", 0) * x.get("ms", 0) for x in step) / max(tot("ms"), 1e-9),
             "issue_slots_busy": sum(x.get("issue", 0) * x.get("ms", 0) for x in step) / max(tot("ms"), 1e-9) / 100,
             "achieved_occupancy": sum(x.get("occ", 0) * x.get("ms", 0) for x in step) / max(tot("ms"), 1e-9) / 100,
             "l2_hit_rate": sum(x.get("l2hit", 0) * x.get("ms", 0) for x in step) / max(tot("ms"), 1e-9) / 100,
             "l2_atom_sectors": tot("atom"), "l2_red_sectors": tot("red"), "sm_mhz": 1965.0}
        table.append(e)
        lines.append(f"{name:12s} {label:24s} {per_step} launch(es) {tot('ms'):8.2f} ms  DRAM {dram / 1e9:7.2f} GB "
                     f"({dram / 1e9 / max(tot('ms') / 1e3, 1e-9):7.1f} GB/s)  {tot('inst') / 1e9:6.2f} G warp-inst  "
                     f"IPC {e['ipc']:.2f}  issue {100 * e['issue_slots_busy']:.0f}%  occ {100 * e['achieved_occupancy']:.0f}%"
                     f"  L2 hit {100 * e['l2_hit_rate']:.0f}%  atom {tot('atom') / 1e6:.1f} M  red {tot('red') / 1e6:.1f} M")
    # keep the entries (and summary lines) of kernels this capture set did not re-measure
    jpath = os.path.join(os.path.dirname(prefix) or ".", "roofline_traffic.json")
    spath = f"{prefix}_ncu_summary.txt"
    got = {(e["config"], e["kernel"]) for e in table}
    if os.path.exists(jpath):
        for e in json.load(open(jpath)):
            if (e.get("config"), e.get("kernel")) not in got:
                table.append(e)
    if os.path.exists(spath):
        names = {ln.split()[0] for ln in lines}
        for ln in open(spath).read().splitlines():
            if ln and not ln.startswith("#") and ln.split()[0] not in names and ln.split()[0] in SPECS:
                lines.append(ln)
    json.dump(table, open(jpath, "w"), indent=1)
    with open(spath, "w") as f:
        f.write("# r02 ncu --set full captures (scripts/r02b_final.sh), per timed step of bench.py\n")
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
