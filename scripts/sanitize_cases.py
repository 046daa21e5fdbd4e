"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): every
counting tier on C0-sized and adversarial inputs, each checked against the oracle.
  compute-sanitizer --tool racecheck python scripts/sanitize_cases.py [case ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1607_06618_b200 import gerbil  # noqa: E402
from tests.helpers import compare  # noqa: E402

C0 = synth.Workload(seed=1, genome_len=100_000, read_len=100, n_reads=3000, err=0.0025, nrate=0.001)
LONG = synth.Workload(seed=5, genome_len=200_000, read_len=2000, n_reads=60, err=0.01)
ALLA = b"".join(b">a%d\n" % i + b"A" * 300 + b"\n" for i in range(40)) + b">lc\n" + b"ACGT" * 200 + b"\n"

CASES = {
    # name: (text, k, m, min_count, Gerbil kwargs)
    "smem_k40": (lambda: synth.fastx(C0, synth.FASTQ), 40, 15, 1, dict(n_bins=1 << 16)),
    "smem_k65_mc2": (lambda: synth.fastx(C0, synth.FASTQ), 65, 15, 2, dict(n_bins=1 << 16)),
    "smem_alla": (lambda: ALLA, 40, 15, 1, dict(n_bins=1 << 16)),
    "ref_k150": (lambda: synth.fastx(LONG, synth.FASTA), 150, 15, 1, dict(n_bins=1 << 16)),
    "ref_alla": (lambda: ALLA, 150, 11, 1, dict(n_bins=4)),
    # GERBIL_REF_DBG=16 (zero fingerprints): every occupied slot met is verified, the deferred
    # queue and the re-probe after a mismatch run constantly
    "ref_k200_zfp": (lambda: synth.fastx(LONG, synth.FASTA), 200, 15, 2, dict(n_bins=1 << 16)),
    "l2_k28": (lambda: synth.fastx(C0, synth.FASTQ), 28, 7, 1, dict(n_bins=1, count_mode=gerbil.COUNT_L2)),
    "l2_k200": (lambda: synth.fastx(LONG, synth.FASTA), 200, 11, 2, dict(n_bins=16, count_mode=gerbil.COUNT_L2)),
    "l2_overflow": (lambda: synth.fastx(C0, synth.FASTQ), 33, 9, 1,
                    dict(n_bins=4, count_mode=gerbil.COUNT_L2, max_probes=1, target_load=1.6, distinct_ratio=0.3)),
    "l2_overflow_k28": (lambda: synth.fastx(C0, synth.FASTQ), 28, 9, 1,
                        dict(n_bins=4, count_mode=gerbil.COUNT_L2, max_probes=1, target_load=1.6, distinct_ratio=0.3)),
    "l2_overflow_k40_p4": (lambda: synth.fastx(C0, synth.FASTQ), 40, 9, 1,
                           dict(n_bins=4, count_mode=gerbil.COUNT_L2, max_probes=4, target_load=1.2,
                                distinct_ratio=0.3)),
    "l2_k40": (lambda: synth.fastx(C0, synth.FASTQ), 40, 9, 1, dict(n_bins=4, count_mode=gerbil.COUNT_L2)),
}


def run(name):
    text_fn, k, m, mc, kw = CASES[name]
    if name.endswith("_zfp"):
        os.environ["GERBIL_REF_DBG"] = "16"
    else:
        os.environ.pop("GERBIL_REF_DBG", None)
    text = text_fn()
    ref = oracle.count(text, k, mc)
    with gerbil.Gerbil(**kw) as g:
        g.count(k, m, mc, text=text)
        keys, counts = g.fetch(sorted=True)
    compare(keys, counts, k, ref)
    print(f"{name}: ok ({len(ref.kmers)} k-mers)", flush=True)


if __name__ == "__main__":
    for n in (sys.argv[1:] or list(CASES)):
        run(n)
