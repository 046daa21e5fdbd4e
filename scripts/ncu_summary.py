"""Summarise an .ncu-rep (details + stall reasons + key raw metrics) as text."""
import csv, subprocess, sys, io

def page(rep, p):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))

def main(rep):
    rows = page(rep, "details")
    want = {"Duration", "DRAM Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput", "Compute (SM) Throughput",
            "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "L2 Hit Rate", "Executed Ipc Active",
            "Grid Size", "Block Size", "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block",
            "Block Limit Registers", "Block Limit Shared Mem", "Memory Throughput", "Issue Slots Busy"}
    seen = set()
    for r in rows[1:]:
        if len(r) >= 4 and r[-4] in want and (r[-4], r[-3]) not in seen:
            seen.add((r[-4], r[-3]))
            print(f"  {r[-4]:35s} {r[-2]:>12s} {r[-3]}")
    raw = page(rep, "raw")
    h, v = raw[0], raw[2] if len(raw) > 2 else raw[1]
    d = dict(zip(h, v))
    stalls = {}
    for k2, val in d.items():
        if k2.startswith("smsp__pcsamp_warps_issue_stalled_") and not k2.endswith("not_issued"):
            try:
                stalls[k2.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(val.replace(",", ""))
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1
    top = sorted(stalls.items(), key=lambda x: -x[1])[:8]
    print("  stalls:", ", ".join(f"{n} {100*c/tot:.0f}%" for n, c in top))
    for m in ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
              "lts__t_sectors_srcunit_tex_op_atom.sum", "lts__t_sectors_srcunit_tex_op_red.sum",
              "lts__t_sectors_srcunit_tex_op_write.sum", "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
              "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct",
              "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
              "gpu__time_duration.sum"]:
        if m in d:
            print(f"  {m:55s} {d[m]} {raw[1][h.index(m)] if len(raw)>2 else ''}")

if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print("==", rep)
        main(rep)
