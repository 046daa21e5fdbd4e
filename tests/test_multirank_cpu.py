"""N > 1 host logic on CPU: world_size-2 (and 3) process groups over gloo.

Every rank builds its own per-bin step-(b) histogram (seeded by rank, skewed like
minimizer bins), all-gathers it with torch.distributed (gloo, 127.0.0.1), and calls
the library's host-only exchange plan (gerbil_exchange_plan, the code the NCCL path
runs before its all-to-all). Checked across ranks: identical owner maps; every bin
owned by exactly one rank (PAPER.md:49 — all occurrences of a k-mer in one temporary
file, hence on one GPU); each rank's send sizes to d equal d's receive sizes from
it (the all-to-all is consistent); everything sent is received; LPT balance
(max load <= mean + heaviest bin).
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.distributed as dist


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _hist(rank: int, n_bins: int) -> np.ndarray:
    rng = np.random.default_rng(1000 + rank)
    sm = rng.poisson(rng.gamma(2.0, 20.0, n_bins)).astype(np.uint64)      # super-mers per bin
    win = sm * rng.integers(5, 30, n_bins).astype(np.uint64)               # windows
    words = sm * rng.integers(2, 4, n_bins).astype(np.uint64)              # payload words
    if n_bins > 7:
        win[7] *= np.uint64(50)                                            # one heavy bin
    return np.stack([win, sm, words])


def _worker(rank: int, world: int, port: int, n_bins: int, out: str) -> None:
    """One rank (own process): all-gather histograms, plan, all-gather plans; rank 0 saves."""
    import torch

    from paper_1607_06618_b200 import gerbil

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = torch.from_numpy(_hist(rank, n_bins).astype(np.int64))
        parts = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine)
        H = np.stack([p.numpy().astype(np.uint64) for p in parts])
        plan = gerbil.exchange_plan(H, rank)
        t = torch.from_numpy(np.concatenate([plan.owner.astype(np.int64), plan.send_desc_off.astype(np.int64),
                                             plan.send_word_off.astype(np.int64),
                                             plan.recv_desc_off.astype(np.int64),
                                             plan.recv_word_off.astype(np.int64)]))
        allp = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allp, t)
        if rank == 0:
            np.savez(out, H=H, plans=np.stack([a.numpy() for a in allp]))
    finally:
        dist.destroy_process_group()


def _run(world: int, n_bins: int, tmp_path):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "plan.npz")
    port = _free_port()
    code = "import sys; from tests.test_multirank_cpu import _worker; _worker(*map(int, sys.argv[1:5]), sys.argv[5])"
    env = {**os.environ, "PYTHONPATH": root + os.pathsep + os.environ.get("PYTHONPATH", "")}
    procs = [subprocess.Popen([sys.executable, "-c", code, str(r), str(world), str(port), str(n_bins), out],
                              cwd=root, env=env) for r in range(world)]
    for p in procs:
        assert p.wait(timeout=300) == 0
    z = np.load(out)
    return z["H"], list(z["plans"])


# (2, 4096): the group-level plan of the device-planned multi-GPU path — 2^22 bins exchanged as
# 4096 groups of 1024 bins (waves.cu exchange_groups runs exchange_plan over group histograms)
@pytest.mark.parametrize("world,n_bins", [(2, 512), (2, 1), (3, 97), (2, 4096), (3, 4096)])
def test_exchange_plan_consistent_across_gloo_ranks(world, n_bins, tmp_path):
    H, plans = _run(world, n_bins, tmp_path)
    P, B = world, n_bins
    owners = [p[:B] for p in plans]
    for o in owners[1:]:
        assert np.array_equal(o, owners[0]), "ranks disagree on bin owners"
    owner = owners[0]
    assert owner.min() >= 0 and owner.max() < P
    W = P + 1
    sd = [p[B:B + W] for p in plans]
    sw = [p[B + W:B + 2 * W] for p in plans]
    rd = [p[B + 2 * W:B + 3 * W] for p in plans]
    rw = [p[B + 3 * W:B + 4 * W] for p in plans]
    for s in range(P):
        for d in range(P):
            # what s sends to d == what d receives from s, from both sides' own arithmetic
            assert sd[s][d + 1] - sd[s][d] == rd[d][s + 1] - rd[d][s]
            assert sw[s][d + 1] - sw[s][d] == rw[d][s + 1] - rw[d][s]
            expect = H[s, 1][owner == d].sum()
            assert sd[s][d + 1] - sd[s][d] == expect
    total_sm = int(H[:, 1].sum())
    assert sum(int(rd[d][P]) for d in range(P)) == total_sm == sum(int(sd[s][P]) for s in range(P))
    # each rank's data lands, in d's receive buffer, after the lower ranks' (the receive base the
    # group exchange computes on the sending side)
    for d in range(P):
        for s in range(P):
            assert rw[d][s] == sum(int(sw[q][d + 1] - sw[q][d]) for q in range(s))
    # LPT balance on windows
    gw = H[:, 0].sum(axis=0).astype(np.float64)
    load = np.array([gw[owner == d].sum() for d in range(P)])
    assert load.max() <= load.mean() + gw.max() + 1e-9


def test_exchange_plan_usage_errors():
    from paper_1607_06618_b200 import gerbil

    H = np.zeros((2, 3, 4), np.uint64)
    with pytest.raises(gerbil.GerbilError):
        gerbil.exchange_plan(H, 2)
    with pytest.raises(gerbil.GerbilError):
        gerbil.exchange_plan(np.zeros((2, 3, 0), np.uint64), 0)
