"""Benchmark of the B200 Gerbil counting phase.

A step = one pass of the whole hot path (b) minimizer/super-mer/bin → (c) bin
shuffle → (d) per-bin counting → (e) min-count compaction, over one batch of
synthetic reads already resident in HBM, through the C ABI
(gerbil_count_device). N=1 workload = BASELINE.json configs[1]: F. vesca-scale
synthetic Illumina reads (5×10^7 × 100 bp = 5 Gbp), k=40, min_count=1; m=15 (results do
not depend on m; m=15 makes ~4M bins small enough for the shared-memory count kernel).
Under torchrun (N>1) every rank counts its own 5 Gbp shard (weak scaling) and
bins are shuffled across ranks with NCCL.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Rank 0 prints ONE JSON line. `--impl reference` times the CPU oracle (the
reference arm of this tier) on the host cores instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "input bases/s counted (k-mer counting phase, steps b-e)"
UNIT = "bases/s"

# configs[1]: "F. vesca-scale synthetic Illumina reads (~5 Gbp, 100-bp), k=40, 1xB200"
C1 = dict(seed=2, genome_len=240_000_000, read_len=100, n_reads=50_000_000, err=0.0033, nrate=0.0001)
K, M, MIN_COUNT = 40, 15, 1
WORKLOAD_NAME = ""


def set_m(m: int) -> None:
    global M, WORKLOAD_NAME
    M = m
    WORKLOAD_NAME = (f"C1: F. vesca-scale synthetic Illumina reads, 5e7 x 100 bp = 5 Gbp per GPU, k=40, m={m}, "
                     "min_count=1")


set_m(M)
ORACLE_SAMPLE_READS = 100_000  # 10 Mbp per oracle step: ~10 s of single-thread std::map work


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _cpu_info():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return model, os.cpu_count() or 1


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def run_reference(args) -> None:
    """Reference arm: the CPU oracle as it stands, on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    import synth

    w = synth.Workload(**{**C1, "n_reads": ORACLE_SAMPLE_READS})
    text = synth.fastx(w, synth.FASTQ)
    for _ in range(args.warmup):
        oracle.count(text, K, MIN_COUNT)
    times = []
    windows = 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r = oracle.count(text, K, MIN_COUNT)
        times.append(time.perf_counter() - t0)
        windows = r.windows
    t = statistics.median(times)
    value = w.n_bases / t
    model, ncpu = _cpu_info()
    sample = f"first {ORACLE_SAMPLE_READS} reads of C1 ({w.n_bases / 1e6:.0f} Mbp) per step, FASTQ text, single thread"
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "string keys (std::map)", "data": "synthetic",
        "config": {"workload": WORKLOAD_NAME, "k": K, "m": M, "min_count": MIN_COUNT, "sample": sample},
        "kmers_per_s": windows / t,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                         "cpu": model, "host_cores": ncpu},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def cpu_baseline() -> dict:
    import oracle
    import synth

    w = synth.Workload(**{**C1, "n_reads": ORACLE_SAMPLE_READS})
    text = synth.fastx(w, synth.FASTQ)
    t0 = time.perf_counter()
    r = oracle.count(text, K, MIN_COUNT)
    t = time.perf_counter() - t0
    model, ncpu = _cpu_info()
    return {"value": w.n_bases / t, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"first {ORACLE_SAMPLE_READS} reads of C1 ({w.n_bases / 1e6:.0f} Mbp), k={K}, "
                      f"single-thread std::map oracle, {t:.1f} s", "kmers_per_s": r.windows / t,
            "cpu": model, "host_cores": ncpu}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--reads", type=int, default=C1["n_reads"], help="reads per GPU (default: C1)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--table-mb", type=int, default=0)
    ap.add_argument("--bins", type=int, default=0)
    ap.add_argument("--m", type=int, default=M, help="minimizer length (results are invariant in m)")
    ap.add_argument("--count-mode", type=int, default=0, help="gerbil_config.count_mode (0 auto, 1 L2, 2 smem)")
    args = ap.parse_args()
    set_m(args.m)
    if args.impl == "reference":
        run_reference(args)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    from paper_1607_06618_b200 import gerbil

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream(dev)

    uid = None
    if world > 1:
        obj = [gerbil.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    # N > 1: ranks need the same explicit B; the multi-rank plan (LPT over all bins) runs on the
    # host, so keep B moderate there (L2 wave tables); N = 1 lets the library pick (4M bins, m = 15)
    n_bins = args.bins or (4096 if world > 1 else 0)
    g = gerbil.Gerbil(device=local, rank=rank, world=world, unique_id=uid, n_bins=n_bins,
                      stream=stream.cuda_stream, timing=True,
                      wave_table_bytes=args.table_mb << 20, count_mode=args.count_mode)

    w = synth.Workload(**{**C1, "n_reads": args.reads, "first_read": rank * args.reads})
    codes, nmask, rs = synth.packed_device(w, device=dev, stream=stream.cuda_stream)
    torch.cuda.synchronize(dev)

    def step():
        g.count_device(codes, nmask, rs, w.n_reads, K, M, MIN_COUNT)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize(dev)

    sampler = ClockSampler(local)
    sampler.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    per_kernel = {"count": [0.0, 0], "compact": [0.0, 0], "supermer": [0.0, 0], "shuffle": [0.0, 0],
                  "smem": [0.0, 0]}
    launches = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
        st = g.stats()
        per_kernel["count"][0] += st["ms_count"]
        per_kernel["count"][1] += st["launches_count"]
        per_kernel["compact"][0] += st["ms_compact"]
        per_kernel["compact"][1] += st["launches_compact"]
        per_kernel["supermer"][0] += st["ms_supermer"]
        per_kernel["shuffle"][0] += st["ms_shuffle"]
        per_kernel["smem"][0] += st["ms_smem"]
        per_kernel["smem"][1] += st["launches_smem"]
        launches += st["launches_total"]
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    st = g.stats()
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        tot = torch.tensor([float(st["input_bases"]), float(st["valid_windows"])], device=dev,
                           dtype=torch.float64)
        dist.all_reduce(tot)
        total_bases, total_windows = float(tot[0]), float(tot[1])
    else:
        total_bases, total_windows = float(st["input_bases"]), float(st["valid_windows"])
    value = total_bases / (ms / 1e3)

    # ---- roofline of the dominant kernel (count, step d) ----------------------------------
    peak, peak_src = _peaks()
    W = st["W"]
    sm_bases = st["valid_windows"] + st["supermers"] * (K - 1)
    traffic_tbl = {}
    tpath = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(tpath):
        tj = json.load(open(tpath))
        for e in (tj if isinstance(tj, list) else [tj]):
            if e.get("workload") == WORKLOAD_NAME:
                traffic_tbl[e.get("kernel")] = e
    smem_share = st["smem_windows"] / max(st["valid_windows"], 1)
    if smem_share >= 0.5:
        # step (d)+(e) in per-warp shared-memory tables (count_smem.cu): per window, the
        # algorithmic HBM bytes are the descriptor (8 B/super-mer) and packed bases (0.25 B/base)
        # it reads and the (8W+4)-byte (k-mer, count) pair it writes per kept k-mer; the table
        # lives in shared memory. Units per launch = the windows it counted.
        n_smem = max(per_kernel["smem"][1], 1)
        avg_ms = per_kernel["smem"][0] / n_smem
        per_window = (8 * st["supermers"] + 0.25 * sm_bases + (8 * W + 4) * st["kept"]) / max(st["valid_windows"], 1)
        bytes_per_launch = per_window * st["smem_windows"] / max(st["launches_smem"], 1)
        achieved = bytes_per_launch / (avg_ms / 1e3) / 1e9 if avg_ms > 0 else None
        kname = "count_smem_kernel<2,true>"
        tr = traffic_tbl.get("count_smem_kernel", {})
        roofline = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": (achieved / peak) if achieved else None,
                    "traffic": tr.get("dram_bytes_per_launch"), "peak_source": peak_src,
                    "bytes_model": f"per window: (8*supermers + 0.25*supermer_bases + {8 * W + 4}*kept) / windows; "
                                   "x windows counted in shared memory per launch",
                    "algorithmic_bytes_per_launch": bytes_per_launch, "avg_launch_ms": avg_ms,
                    "launches_per_step": st["launches_smem"],
                    "share_of_step": per_kernel["smem"][0] / args.steps / ms,
                    "windows_share": smem_share,
                    "issue_slot_util": tr.get("issue_slots_busy"),
                    "note": "table in shared memory: the kernel is bound by instruction issue and "
                            "shared-memory latency (ncu issue_slot_util), not HBM; DESIGN.md §4"}
    else:
        # table bytes per slot: 16 B inline slots for k <= 46, else the chunked bucket / 4
        slot = 16 if K <= 46 else (32 + 32 * ((K + 30) // 31)) / 4
        n_count = max(per_kernel["count"][1], 1)
        avg_count_ms = per_kernel["count"][0] / n_count
        # algorithmic bytes per step of the count kernel (SURVEY.md §8(d) stream model restricted to
        # this kernel): descriptors (8 B/super-mer), packed super-mer bases
        # (0.25 B/base), and one write of every claimed table slot (slot B per distinct k-mer).
        count_bytes_step = 8 * st["supermers"] + 0.25 * sm_bases + slot * st["distinct"]
        bytes_per_launch = count_bytes_step / max(st["launches_count"], 1)
        achieved = bytes_per_launch / (avg_count_ms / 1e3) / 1e9 if avg_count_ms > 0 else None
        tr = traffic_tbl.get("count_inline_kernel", {})
        roofline = {"bound": "hbm", "kernel": "count_inline_kernel<2,true>", "achieved": achieved, "peak": peak,
                    "unit": "GB/s", "frac": (achieved / peak) if achieved else None,
                    "traffic": tr.get("dram_bytes_per_launch"), "peak_source": peak_src,
                    "bytes_model": f"8*supermers + 0.25*supermer_bases + {slot:g}*distinct per step",
                    "algorithmic_bytes_per_launch": bytes_per_launch,
                    "avg_launch_ms": avg_count_ms, "launches_per_step": st["launches_count"],
                    "share_of_step": per_kernel["count"][0] / args.steps / ms,
                    "note": "L2-resident table: the kernel is bound by the L2 random-access rate of its "
                            "bucket-load + atomic pattern, not HBM; see l2_ceiling and DESIGN.md §4"}
        # The bound that applies: one 64-byte bucket load + one atomic into the same bucket per window
        # (RED for a k-mer already present, 128-bit CAS for a new one). scripts/l2_micro.cu measured
        # what B200's L2 sustains for these patterns on a 64 MiB table (profiles/r01_l2_micro.txt).
        L2_LOAD_RED, L2_LOAD_CAS = 49.2e9, 38.3e9  # ops/s, "load+red" / "load+cas" rows
        new_k = float(st["distinct"])
        hits = max(float(st["valid_windows"]) - new_k, 0.0)
        t_floor = hits / L2_LOAD_RED + new_k / L2_LOAD_CAS
        d_ms = per_kernel["count"][0] / args.steps  # steps (d)+(e) device time per step
        roofline["l2_ceiling"] = {
            "bound": "l2_random_ops", "unit": "G window-ops/s",
            "achieved": float(st["valid_windows"]) / (d_ms / 1e3) / 1e9 if d_ms > 0 else None,
            "peak": float(st["valid_windows"]) / t_floor / 1e9 if t_floor > 0 else None,
            "frac": (t_floor * 1e3 / d_ms) if d_ms > 0 else None,
            "floor_ms": t_floor * 1e3, "measured_ms": d_ms,
            "source": "profiles/r01_l2_micro.txt (load+red 49.2, load+cas 38.3 Gop/s, 64 MiB table); "
                      "measured_ms = steps (d)+(e) incl. compaction"}

    # ---- end to end through the C ABI with host buffers -----------------------------------
    e2e = None
    if not args.no_e2e and args.e2e_steps > 0:
        hc = torch.empty(codes.numel(), dtype=torch.int64, pin_memory=True)
        hn = torch.empty(nmask.numel(), dtype=torch.int64, pin_memory=True)
        hr = torch.empty(rs.numel(), dtype=torch.int64, pin_memory=True)
        hc.copy_(codes)
        hn.copy_(nmask)
        hr.copy_(rs)
        # size the record stream once (a full untimed call), then stream into pinned memory
        try:
            need = g.count_host_stream(hc.numpy(), hn.numpy(), hr.numpy(), w.n_reads, K, M, MIN_COUNT, out=None)
        except gerbil.GerbilError as e:
            need = e.needed_bytes
        rec = torch.empty(int(need * 1.02) + (1 << 20), dtype=torch.uint8, pin_memory=True).numpy()
        h2d = d2h = 0
        times = []
        for i in range(args.e2e_steps + 1):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            nbytes = g.count_host_stream(hc.numpy(), hn.numpy(), hr.numpy(), w.n_reads, K, M, MIN_COUNT, out=rec)
            dt = time.perf_counter() - t0
            if i > 0:
                times.append(dt)
            h2d = (hc.numel() + hn.numel() + hr.numel()) * 8
            d2h = nbytes
        est = g.stats()
        te = max(times) if times else float("nan")
        if world > 1:
            t = torch.tensor([te], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        e2e = {"value": total_bases / te, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": te * 1e3,
               "stage_ms": {x: est["ms_" + x] for x in ("h2d", "supermer", "shuffle", "count", "compact")},
               "path": "gerbil_count_host_stream: pinned H2D of the packed batch, steps (b)-(e), and every "
                       "(k-mer, count) as the paper's binary record (App. C) streamed to pinned host memory by "
                       "the compaction kernel while later waves are counted; wall clock per call, max over ranks"}

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64 (2-bit packed k-mer words, u32 counts)", "data": "synthetic",
            "config": {"workload": WORKLOAD_NAME, "reads_per_gpu": w.n_reads, "read_len": w.read_len,
                       "genome_len": w.genome_len, "err": w.err, "nrate": w.nrate, "k": K, "m": M,
                       "min_count": MIN_COUNT, "n_bins": st["n_bins"], "waves": st["waves"],
                       "parallelism": f"bins sharded over {world} GPU(s)",
                       "l2": "inputs larger than L2 (packed reads 1.25 GB/GPU); no flush"},
            "kmers_per_s": total_windows / (ms / 1e3),
            "stage_ms": {"supermer": per_kernel["supermer"][0] / args.steps,
                         "shuffle": per_kernel["shuffle"][0] / args.steps,
                         "count": per_kernel["count"][0] / args.steps,
                         "count_smem_kernel": per_kernel["smem"][0] / args.steps,
                         "compact": per_kernel["compact"][0] / args.steps},
            "result": {"distinct": st["distinct"], "kept": st["kept"], "supermers": st["supermers"],
                       "valid_windows": st["valid_windows"], "ratio_observed": st["ratio_observed"],
                       "overflow_kmers": st["overflow_kmers"],
                       "first_probe_frac": st["probe_first"] / max(st["probe_first"] + st["probe_more"], 1),
                       "max_probes": st["probe_max"], "smem_bins": st["smem_bins"],
                       "smem_failed": st["smem_failed"], "smem_windows": st["smem_windows"],
                       "smem_slots": st["smem_slots"]},
            "roofline": roofline,
            "gpu_launches": launches,
            "clocks": clocks,
            "e2e": e2e,
        }
        if not args.no_cpu_baseline and world == 1:
            out["cpu_baseline"] = cpu_baseline()
        print(json.dumps(out), flush=True)
    g.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
